"""Port of the reference's own CPU algorithm for the online answer -- the
timed CPU baseline ("kind": "port"). TEST / BENCH INFRASTRUCTURE ONLY.

The reference is pure Python over numpy/OpenBLAS and gmpy2; it cannot travel
to the GPU box (no /root/reference there, no gmpy2 in the image), so this
module restates its algorithm with the same numerical method and the same
BLAS calls:
  * global hint: two exact float64 GEMMs with A split 16/16
    (protocol.py:195-207)
  * db_matvec: centered float64 GEMV over an (d1, d0) float64 copy of db^T,
    corrected back mod 2^32 (protocol.py:190-193, :242-257)
  * hv = H_scaled . ck_o mod m through the 240 x 27-bit-prime RNS engine:
    16-bit-limb residue conversion against a power table (rns.py:52-86),
    per-prime batched matvecs with a 14-bit split (rns.py:163-188), Garner
    mixed-radix reconstruction and big-int assembly (rns.py:94-145)
  * t = (scaled_b(b) + hv) mod m (protocol.py:259-269, :349-350)
Verified bit-exact against tests/golden by tests/test_ref_port.py.
"""

import numpy as np

SPLIT = 14


def _is_prime(x: int) -> bool:
    if x < 2:
        return False
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if x % p == 0:
            return x == p
    d, s = x - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17):
        y = pow(a, d, x)
        if y in (1, x - 1):
            continue
        for _ in range(s - 1):
            y = y * y % x
            if y == x - 1:
                break
        else:
            return False
    return True


class Basis:
    """The `count` largest primes below 2^bits, descending (rns.py:32-49)."""

    def __init__(self, bits=27, count=240):
        primes = []
        x = (1 << bits) - 1
        while len(primes) < count:
            if _is_prime(x):
                primes.append(x)
            x -= 1
        self.primes = primes
        self.p_f = np.array(primes, dtype=np.float64)
        self.p_i = np.array(primes, dtype=np.int64)
        self.count = count
        inv = np.zeros(count, dtype=np.int64)
        Q = 1
        for i, p in enumerate(primes):
            inv[i] = pow(Q % p, -1, p) if i else 1
            Q *= p
        self.Q = Q
        self.inv_partial = inv
        self._consts = {}

    def power_table(self, nlimbs):
        tbl = np.empty((nlimbs, self.count), dtype=np.float64)
        cur = np.ones(self.count, dtype=np.int64)
        for k in range(nlimbs):
            tbl[k] = cur
            cur = (cur << 16) % self.p_i
        return tbl

    def to_rns(self, values) -> np.ndarray:
        values = [int(v) for v in values]
        maxbits = max((v.bit_length() for v in values), default=0)
        nbytes = max(2, ((maxbits + 15) // 16) * 2)
        buf = b"".join(v.to_bytes(nbytes, "little") for v in values)
        limbs = np.frombuffer(buf, dtype="<u2").reshape(len(values), nbytes // 2).astype(np.float64)
        tbl = self.power_table(limbs.shape[1])
        step = 1 << (53 - 16 - 27)
        acc = np.zeros((len(values), self.count), dtype=np.float64)
        for s in range(0, limbs.shape[1], step):
            acc = np.mod(acc + limbs[:, s:s + step] @ tbl[s:s + step], self.p_f)
        return acc

    def assembly(self, mod):
        c = self._consts.get(mod)
        if c is None:
            c, run = [], 1
            for p in self.primes:
                c.append(run % mod)
                run *= p
            self._consts[mod] = c
        return c

    def from_rns_mod(self, res, mod) -> list:
        """Garner digits vectorised across rows, then assembly mod `mod`."""
        res = np.asarray(res, dtype=np.int64)
        nrows = res.shape[0]
        ip = self.p_i
        digits = np.zeros((self.count, nrows), dtype=np.int64)
        acc = np.zeros((self.count, nrows), dtype=np.int64)
        pm = np.ones(self.count, dtype=np.int64)
        for k in range(self.count):
            pk = int(ip[k])
            d = (res[:, k] - acc[k]) % pk
            d = d * int(self.inv_partial[k]) % pk
            digits[k] = d
            if k + 1 < self.count:
                acc = (acc + pm[:, None] * d[None, :]) % ip[:, None]
                pm = pm * pk % ip
        consts = self.assembly(mod)
        out = []
        for r in range(nrows):
            v = 0
            col = digits[:, r]
            for k in range(self.count):
                dk = int(col[k])
                if dk:
                    v += dk * consts[k]
            out.append(v % mod)
        return out


class PortState:
    """Server state built the reference's way for db (d0, d1) uint8.

    For d0 <= 32768 this is exactly the reference's fast path (the float64
    exactness bound d0 * 128 * 2^31 <= 2^53, protocol.py:177-179). Beyond it
    (BASELINE configs[2], d0 = 92682, where the reference falls to its
    Python triple loops, protocol.py:209-217 / :253-257) the same float64
    GEMMs / GEMV run over d0 chunks of <= 32768 records and the chunk results
    are summed mod 2^32 -- the "chunked restatement" of SURVEY 8c."""

    CHUNK = 32768

    def __init__(self, db, A, cap, basis=None):
        db = np.asarray(db)
        self.d0, self.d1 = db.shape
        self.cap = cap
        self.groups = -(-self.d1 // cap)
        self.basis = basis or Basis()
        Ai = np.asarray(A, dtype=np.int64)
        mask = (1 << 32) - 1
        h = np.zeros((self.d1, Ai.shape[1]), dtype=np.int64)
        for s0 in range(0, self.d0, self.CHUNK):
            s1 = min(self.d0, s0 + self.CHUNK)
            dbt = db[s0:s1].astype(np.float64).T
            glo = (dbt @ (Ai[s0:s1] & 0xFFFF).astype(np.float64)).astype(np.int64)
            ghi = (dbt @ (Ai[s0:s1] >> 16).astype(np.float64)).astype(np.int64)
            h = (h + np.mod(glo, 1 << 32) + (np.mod(ghi, 1 << 16) << 16)) & mask
            del dbt, glo, ghi
        self.H = ((1 << 32) - h) & mask
        n = self.H.shape[1]
        scaled = []
        for g in range(self.groups):
            blk = np.ascontiguousarray(self.H[g * cap:(g + 1) * cap].astype("<u4").T)
            scaled.append([int.from_bytes(blk[i].tobytes(), "little") for i in range(n)])
        flat = [x for row in scaled for x in row]
        res = self.basis.to_rns(flat)
        self.H_rns = np.ascontiguousarray(res.T.reshape(self.basis.count, self.groups, n))
        self._chunks = []
        for s0 in range(0, self.d0, self.CHUNK):
            s1 = min(self.d0, s0 + self.CHUNK)
            part = db[s0:s1]
            self._chunks.append((s0, s1, (part.astype(np.float64) - 128.0).T.copy(),
                                 (part.astype(np.int64) - 128).sum(axis=0)))

    def db_matvec(self, qu):
        total = np.zeros(self.d1, dtype=np.int64)
        for s0, s1, dbt_c, colsum_c in self._chunks:
            q = qu[s0:s1]
            quf = q.astype(np.float64) - float(1 << 31)
            s = (dbt_c @ quf).astype(np.int64)
            sum_quc = int(q.astype(np.uint64).sum()) - (s1 - s0) * (1 << 31)
            part = s + (colsum_c << 31) + (128 * sum_quc + (s1 - s0) * 128 * (1 << 31))
            total = np.mod(total + np.mod(part, 1 << 32), 1 << 32)
        return total.astype(np.uint64)

    def rns_matvec(self, v, m):
        b = self.basis
        vint = b.to_rns(v).astype(np.int64)
        vlo = (vint & ((1 << SPLIT) - 1)).astype(np.float64)
        vhi = (vint >> SPLIT).astype(np.float64)
        lo = self.H_rns @ vlo.T[:, :, None]
        hi = self.H_rns @ vhi.T[:, :, None]
        p = b.p_f[:, None]
        t = np.mod(np.mod(lo[:, :, 0], p) + np.mod(hi[:, :, 0], p) * float(1 << SPLIT), p)
        return b.from_rns_mod(t.T, m)

    def respond_t(self, qu, ck_o, m):
        b = self.db_matvec(qu)
        hv = self.rns_matvec(ck_o, m)
        arr = b.astype("<u4")
        bs = [int.from_bytes(arr[g * self.cap:(g + 1) * self.cap].tobytes(), "little")
              for g in range(self.groups)]
        return [(bs[g] + hv[g]) % m for g in range(self.groups)]
