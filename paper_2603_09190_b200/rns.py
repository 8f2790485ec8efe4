"""The reference's residue-number-system API (rns.py:19-188) on the device path.

The B200 answer never needs residues: it reads the global hint H in place
and computes hv = H_scaled . ck_o mod m exactly with integer kernels
(answer.cu, umma_gemm.cu). This module keeps the reference's entry points
for callers that use them directly:

  build_basis(prime_bits, count)  the `count` largest primes < 2^prime_bits,
                                  descending (rns.py:32-49), same RnsBasis
  check_matmul_bound(...)         the exactness check (rns.py:157-160)
  matrix_to_rns(basis, H)         an RnsMatrix: H kept as device limb rows;
                                  np.asarray() gives the reference's
                                  (count, rows, cols) float64 residues,
                                  computed on the device (zpir_rns_residues)
  rns_matmul_mod(basis, H_rns, v, m, h_bound=None)
                                  (H . v) mod m (rns.py:163-188) with the same
                                  ValueErrors, on the device: the answer's
                                  compression kernels with b = 0
ServerGlobalState.H_rns is an RnsMatrix view of the state's device H.
"""

from dataclasses import dataclass

import numpy as np
import torch

SPLIT_BITS = 14


@dataclass
class RnsBasis:
    primes: np.ndarray  # float64, each < 2^27
    Q: int
    inv_partial: np.ndarray  # (prod_{j<i} p_j)^-1 mod p_i
    primes_int: list

    @property
    def count(self):
        return len(self.primes)


def _is_prime_small(x: int) -> bool:
    """Deterministic Miller-Rabin for x < 3.3e9 (bases 2, 3, 5, 7)."""
    if x < 2:
        return False
    for p in (2, 3, 5, 7):
        if x % p == 0:
            return x == p
    d, s = x - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7):
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


def build_basis(prime_bits: int, count: int) -> RnsBasis:
    if prime_bits < 2 or prime_bits > 27:
        raise ValueError("prime size must be between 2 and 27 bits")
    primes = []
    x = (1 << prime_bits) - 1
    while len(primes) < count and x >= 2:
        if _is_prime_small(x):
            primes.append(x)
        x -= 1
    if len(primes) < count:
        raise ValueError("not enough primes of %d bits" % prime_bits)
    Q = 1
    inv = np.zeros(count, dtype=np.int64)
    for i, p in enumerate(primes):
        inv[i] = pow(Q % p, -1, p) if i else 1
        Q *= p
    return RnsBasis(np.array(primes, dtype=np.float64), Q, inv, list(primes))


def check_matmul_bound(basis: RnsBasis, n: int, h_bound: int, v_bound: int):
    if basis.Q <= n * h_bound * v_bound:
        raise ValueError("basis product too small for exact reconstruction")


class RnsMatrix:
    """A big-integer matrix in the reference's residue form, kept on the
    device as 32-bit words: entry (g, k) = sum_j 2^(32 stride j) S[g cap + j][k]
    over the `rows` valid rows of S (rows x n u32; gamma = 2^(32 stride), or
    the general batch scale of a state's layout). Array access
    (np.asarray, shape, indexing) materialises the (count, groups, n) float64
    residues on the device once."""

    def __init__(self, basis, S, rows, cap, groups, gamma=1 << 32, state=None, hbound=None):
        self.basis = basis
        self.S = S
        self.rows, self.cap, self.groups, self.gamma = rows, cap, groups, gamma
        self.n = S.shape[1]
        self.state = state
        self.hbound = hbound      # an upper bound of every entry (exclusive)
        self._res = None

    @property
    def shape(self):
        return (self.basis.count, self.groups, self.n)

    def residues(self) -> np.ndarray:
        if self._res is None:
            from . import _lib
            b = self.basis
            dev = self.S.device
            w = np.empty((b.count, self.cap), dtype=np.uint64)
            for i, p in enumerate(b.primes_int):
                step = self.gamma % p
                acc = 1
                for j in range(self.cap):
                    w[i, j] = acc
                    acc = acc * step % p
            pr = torch.from_numpy(np.array(b.primes_int, dtype=np.uint32).view(np.int32)).to(dev)
            wd = torch.from_numpy(w.view(np.int64)).to(dev)
            out = torch.empty(self.shape, dtype=torch.float64, device=dev)
            st = torch.cuda.current_stream(dev)
            _lib.call("zpir_rns_residues", _lib.ptr(self.S), self.rows, self.n, self.cap,
                      1, _lib.ptr(pr), _lib.ptr(wd), b.count, self.groups,
                      _lib.ptr(out), st.cuda_stream)
            self._res = out.cpu().numpy()
        return self._res

    def __array__(self, dtype=None, copy=None):
        r = self.residues()
        return r.astype(dtype) if dtype is not None else r

    def __getitem__(self, idx):
        return self.residues()[idx]

    def __len__(self):
        return self.basis.count


def matrix_to_rns(basis: RnsBasis, H, device=None) -> RnsMatrix:
    """Residues of a big-integer matrix (rns.py:148-154), held on the device."""
    from . import device as zdev
    from .bigint import ints_to_limbs
    rows = len(H)
    cols = len(H[0]) if rows else 0
    flat = [int(x) for row in H for x in row]
    if any(x < 0 for x in flat):
        raise ValueError("matrix entries must be nonnegative")
    maxbits = max((x.bit_length() for x in flat), default=0)
    L = max(1, -(-maxbits // 32))
    dev = zdev.require_cuda(device)
    limbs = ints_to_limbs(flat, L).reshape(rows, cols, L) if rows and cols else \
        np.zeros((rows, cols, L), dtype=np.uint32)
    S = np.ascontiguousarray(limbs.transpose(0, 2, 1)).reshape(rows * L, cols)
    pad = -(-max(rows * L, 1) // 32) * 32        # answer_rows tiles rows by 32
    Sd = torch.zeros((pad, max(cols, 1)), dtype=torch.int32, device=dev)
    if rows and cols:
        Sd[: rows * L, :cols] = torch.from_numpy(S.view(np.int32)).to(dev)
    return RnsMatrix(basis, Sd[:, :cols] if cols else Sd, rows * L, L, rows,
                     hbound=1 << max(maxbits, 1))


def rns_matmul_mod(basis: RnsBasis, H_rns, v, m: int, h_bound=None) -> list:
    """(H . v) mod m for H in residue form (rns.py:163-188), on the device.
    Same checks and ValueErrors as the reference; the result is exact."""
    from . import device as zdev
    from .bigint import ints_to_limbs, key_ctx, limbs_to_ints
    if not isinstance(H_rns, RnsMatrix):
        raise NotImplementedError("rns_matmul_mod takes the RnsMatrix of matrix_to_rns / "
                                  "ServerGlobalState.H_rns (residue arrays from elsewhere are "
                                  "not reconstructed on this path)")
    count, d, n = H_rns.shape
    if len(v) != n:
        raise ValueError("dimension mismatch")
    v = [int(x) for x in v]
    check_matmul_bound(basis, n, m - 1 if h_bound is None else h_bound, max(v, default=0))
    if n * ((1 << SPLIT_BITS) - 1) * ((1 << 27) - 1) >= 1 << 53:
        raise ValueError("dimension too large for the exact float64 kernel")
    if d == 0:
        return []
    st = H_rns.state
    dev = H_rns.S.device
    stream = torch.cuda.current_stream(dev)
    kctx = key_ctx(m, dev)
    vm = [x % m for x in v]
    cko = torch.from_numpy(ints_to_limbs(vm, kctx.lm).view(np.int32)).to(dev)
    if st is not None:
        lay = st.layout
        b0 = torch.zeros((lay.rows,), dtype=torch.int32, device=dev)
        z = (st.compress_rows(cko, kctx.lm, stream) if st.engine == "umma"
             and kctx.lm in zdev.UMMA_NB and lay.n % 4 == 0 else
             zdev.answer_rows(st.H_dev, b0, 0xFFFFFFFF, cko, kctx.lm, stream=stream))
        t = st._group_stage(z, b0, kctx, kctx.lm, stream)
    else:
        rows_p = H_rns.S.shape[0]
        Sfull = H_rns.S if H_rns.S.is_contiguous() else H_rns.S.contiguous()
        b0 = torch.zeros((rows_p,), dtype=torch.int32, device=dev)
        z = zdev.answer_rows(Sfull, b0, 0xFFFFFFFF, cko, kctx.lm, stream=stream)
        t = zdev.answer_general(z, b0, 0xFFFFFFFF, H_rns.rows, H_rns.cap, d, kctx, 1 << 32,
                                kctx.lm, stream=stream)
    stream.synchronize()
    return limbs_to_ints(t[:d, : kctx.lm].cpu().numpy().view(np.uint32))
