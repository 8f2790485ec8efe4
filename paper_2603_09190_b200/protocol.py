"""ZipPIR server protocol on the B200 path: drop-in for the reference's
ServerGlobalState / hint / respond (protocol.py:159-365).

Same names, argument meaning, return types and exceptions as the reference:
  ServerGlobalState(params, db, basis=None, db_version=0)  ValueError on
      shape / symbol range (protocol.py:166-169)
  hint(state, reg, query_index) -> ClientHint              (protocol.py:291-296)
  respond(state, reg, qmsg, mode=None, timings=None)       ValueError on
      dimensions / mode, KeyError on a missing or stale hint (:337-341),
      timings keys db_matvec / hint_matvec / total (:361-364), COMBINED
      bumps exactly d1' adds and 0 modexp (counters)
Objects from the reference package (ProtocolParams, ClientRegistration,
QueryMessage, ...) are accepted too: only their attributes are read.

Device state per database (built once, swapped whole on update):
  dbt  u8  (rows, ld)  DB = db^T, rows = d1 padded to whole groups and 128,
                       ld = d0 padded to 64  (1 GiB at BASELINE config 2)
  H    u32 (rows, n)   global hint -DB A mod q (128 MiB at config 2)
  A    u32 (ld, lda)   public matrix, kept for incremental row updates
There is no CPU fallback: without the CUDA library or a GPU every entry point
raises.
"""

from dataclasses import dataclass, field
import hashlib
import logging
import threading
import time

import numpy as np
import torch

from . import _lib, counters, device
from .bigint import ints_to_limbs, key_ctx, limbs_to_ints
from .paillier import PaillierCiphertext, PaillierPublicKey, sample_ciphertext  # noqa: F401
from .params import Layout, LweParams, ProtocolParams  # noqa: F401
from .plan import AnswerPlan
from .prg import DOM_CIPHERTEXT_SAMPLE, DOM_PUBLIC_MATRIX

log = logging.getLogger(__name__)

SEPARATE = "separate"
COMBINED = "combined"

# "umma": tcgen05 tensor-core engine (default); "cuda_core": the IDP4A / IMAD
# kernels, for shapes the tensor-core kernels do not take (n % 64 != 0 for the
# hint GEMM, q < 2^32 for the GEMV) and as the second engine the tests compare
ENGINE = "umma"
# SMs given to the compression GEMM while the GEMV streams the DB on the rest
# (both are HBM-bound; H is ~1/8 of the DB bytes; measured optimum, DESIGN 3.2)
COMPRESS_CTAS = 34
# per-client hints: Pippenger bucket updates on the tensor cores (4096-bit m^2)
TC_HINT = True
# transient workspace cap of one tensor-core hint launch (tiles + buckets)
TC_WS_BYTES = 48 * 2**30
# refreshes of at least this many changed DB rows always use the tensor cores; smaller
# ones when the cost model of _tc_refresh_pays says the batch of clients fills the launch
TC_REFRESH_MIN_ROWS = 2048
# full hints: tensor cores when the batch has at least this many exponent rows in total
TC_MIN_ROWS = 2048


@dataclass
class HintRequest:
    pk: PaillierPublicKey
    seed: bytes


@dataclass
class QueryMessage:
    client_id: bytes
    query_index: int
    mode: str
    ck_o: list       # n integers in [0, m)
    qu0: np.ndarray  # d0 integers in [0, q)


@dataclass
class ClientHint:
    query_index: int
    db_version: int
    entries: list    # d1' PaillierCiphertexts
    # device copy of the entries (groups x l2 u32 limbs), kept for COMBINED
    dev: object = field(default=None, repr=False, compare=False)
    # slot decomposition (hint(..., keep_slots=True)): per-DB-row factors
    # W[c] = prod_k ck_r[k]^H[c][k] (Montgomery form) and the fixed-base
    # table P[i][k] = ck_r[k]^(2^(8i)), enabling refresh_hint() after a row
    # update without a full recompute
    slots: object = field(default=None, repr=False, compare=False)
    bases: object = field(default=None, repr=False, compare=False)


@dataclass
class ResponseMessage:
    mode: str
    query_index: int
    t: list
    k: list


@dataclass
class ClientRegistration:
    pk: PaillierPublicKey
    seed: bytes
    client_id: bytes
    hints: dict = field(default_factory=dict)
    consumed: set = field(default_factory=set)


def client_id_of(pk) -> bytes:
    return hashlib.sha256(pk.serialize()).digest()


class _Staging(threading.local):
    """Per-thread pinned host buffers for H2D / D2H staging. Each buffer
    carries the event of the last async copy that read or wrote it; get()
    waits for it, so a buffer is never rewritten while a copy is in flight."""

    def __init__(self):
        self.bufs = {}

    def get(self, key, nbytes):
        ent = self.bufs.get(key)
        if ent is not None:
            ent[1].synchronize()
        if ent is None or ent[0].numel() < nbytes:
            ent = (torch.empty(max(nbytes, 4096), dtype=torch.uint8).pin_memory(),
                   torch.cuda.Event())
            self.bufs[key] = ent
        return ent[0][:nbytes]

    def mark(self, key, stream):
        self.bufs[key][1].record(stream)


_staging = _Staging()


def _h2d(arr: np.ndarray, dev, key, stream) -> torch.Tensor:
    """Host array -> device tensor (same bytes, int32 view for u32 data)."""
    raw = np.ascontiguousarray(arr)
    pinned = _staging.get(key, raw.nbytes)
    pinned.numpy()[:] = raw.view(np.uint8).reshape(-1)
    out = torch.empty(raw.nbytes, dtype=torch.uint8, device=dev)
    with torch.cuda.stream(stream):
        out.copy_(pinned, non_blocking=True)
    _staging.mark(key, stream)
    return out


def _d2h_u32(t: torch.Tensor, key, stream) -> np.ndarray:
    nbytes = t.numel() * 4
    pinned = _staging.get(key, nbytes)
    with torch.cuda.stream(stream):
        pinned.copy_(t.reshape(-1).view(torch.uint8), non_blocking=True)
    stream.synchronize()
    return pinned.numpy().view(np.uint32).reshape(t.shape).copy()


def _host_symbol_check(db: np.ndarray, p: int) -> bool:
    """The reference's range check `db.max() >= p -> ValueError`
    (protocol.py:168-169) without a host pass over a u8 database's bytes:
    every u8 symbol is < 256, so for p >= 256 the check always passes, and for
    p < 256 it runs on the device after the upload (_device_symbol_check).
    Other dtypes are checked here, before the cast to u8. Returns True when
    the device check is still due."""
    if db.dtype == np.uint8:
        return p < 256
    if int(db.max(initial=0)) >= p:
        raise ValueError("database symbol out of range")
    return False


def _device_symbol_check(db_dev: torch.Tensor, p: int) -> None:
    if db_dev.numel() and int(db_dev.max().item()) >= p:
        raise ValueError("database symbol out of range")


class ServerGlobalState:
    """Database-derived state, immutable between update_database calls."""

    def __init__(self, params, db, basis=None, db_version: int = 0, device_=None,
                 engine=None):
        lwe = params.lwe
        db = np.asarray(db)
        if db.shape != (params.d0, params.d1):
            raise ValueError("database shape mismatch")
        dev_check = _host_symbol_check(db, lwe.p)
        self.params = params
        self.db = db
        self.db_version = db_version
        self._basis = basis  # the answer path needs no RNS basis; built lazily for .basis
        lay = self.layout = Layout(params)
        dev = self.device = device.require_cuda(device_)
        stream = torch.cuda.current_stream(dev)
        n, d0, d1 = lay.n, lay.d0, lay.d1
        self._A64 = None
        t0 = time.perf_counter()
        # public matrix A straight from the seeded stream on the device (device ChaCha20)
        self.A_dev = torch.zeros((lay.ld, lay.lda), dtype=torch.int32, device=dev)
        device.chacha_words32(params.a_seed, DOM_PUBLIC_MATRIX, 0, d0, n, self.A_dev, lay.lda,
                              (lay.q - 1) & 0xFFFFFFFF, stream)
        db_dev = device.upload_bytes(db, dev, stream)
        if dev_check:
            _device_symbol_check(db_dev, lwe.p)
        self.dbt = device.transpose_db(db_dev, d0, d1, lay.rows, lay.ld, stream)
        del db_dev
        self.engine = engine or ENGINE
        if self.engine not in ("umma", "cuda_core"):
            raise ValueError(f"unknown engine {self.engine!r}")
        if self.engine == "umma" and n % 64 == 0:
            self.H_dev = device.umma_global_hint(self.dbt, self.A_dev, n, lay.qmask, stream)
        else:
            self.H_dev = device.global_hint(self.dbt, self.A_dev, n, lay.qmask, stream)
        self.H_planes = device.h_planes(self.H_dev, stream) if self.engine == "umma" else None
        stream.synchronize()
        self.hint_time = time.perf_counter() - t0
        self._H_host = None
        self._H_scaled = None
        self._lock = threading.Lock()
        self._tls = threading.local()

    # -- incremental update ------------------------------------------------

    def updated(self, db, db_version: int = None):
        """New state for database `db` built incrementally from this one:
        the DB rows (db columns) that changed are found on the device
        (rows_differ) and only their H rows are recomputed (gather -> hint
        GEMM -> scatter). Returns (new_state, changed_rows). Equivalent to
        ServerGlobalState(params, db, basis, db_version + 1) (server.py:116)."""
        params = self.params
        db = np.asarray(db)
        if db.shape != (params.d0, params.d1):
            raise ValueError("database shape mismatch")
        dev_check = _host_symbol_check(db, params.lwe.p)
        lay = self.layout
        dev = self.device
        stream = torch.cuda.current_stream(dev)
        t0 = time.perf_counter()
        new = object.__new__(ServerGlobalState)
        new.__dict__.update(params=params, db=db, _basis=self._basis, layout=lay, device=dev,
                            engine=self.engine, _A64=self._A64, A_dev=self.A_dev,
                            _H_host=None, _H_scaled=None, _lock=threading.Lock(),
                            _tls=threading.local())
        new.db_version = self.db_version + 1 if db_version is None else db_version
        db_dev = device.upload_bytes(db, dev, stream)
        if dev_check:
            _device_symbol_check(db_dev, params.lwe.p)
        new.dbt = device.transpose_db(db_dev, lay.d0, lay.d1, lay.rows, lay.ld, stream)
        del db_dev
        flags = device.rows_differ(new.dbt, self.dbt, stream)
        changed = np.nonzero(flags[: lay.d1].cpu().numpy())[0].astype(np.int64)
        H = self.H_dev.clone()
        if changed.size:
            R = changed.size
            Rp = -(-R // 128) * 128
            ids = torch.from_numpy(changed.astype(np.int32)).to(dev)
            part = torch.zeros((Rp, lay.ld), dtype=torch.uint8, device=dev)
            device.move_rows(new.dbt, part, ids, scatter=False, stream=stream)
            if self.engine == "umma" and lay.n % 64 == 0:
                Hp = device.umma_global_hint(part, self.A_dev, lay.n, lay.qmask, stream)
            else:
                Hp = device.global_hint(part, self.A_dev, lay.n, lay.qmask, stream)
            device.move_rows(Hp, H, ids, scatter=True, stream=stream)
        new.H_dev = H
        new.H_planes = device.h_planes(H, stream) if self.engine == "umma" else None
        stream.synchronize()
        new.hint_time = time.perf_counter() - t0
        return new, changed

    # -- reference-compatible views (materialised lazily) --------------------

    @property
    def basis(self):
        """The RNS basis (protocol.py:173: build_basis(27, 240) unless given)."""
        if self._basis is None:
            from .rns import build_basis
            self._basis = build_basis(27, 240)
        return self._basis

    @property
    def H_rns(self):
        """H_scaled in residue form (protocol.py:188) as a device-resident view:
        rns.rns_matmul_mod(state.basis, state.H_rns, ck_o, m) runs the answer's
        compression kernels; np.asarray(state.H_rns) gives the reference's
        (count, d1', n) float64 residues (computed on the device)."""
        from .rns import RnsMatrix
        lay = self.layout
        gamma = (1 << (32 * lay.stride)) if lay.stride else lay.gamma
        return RnsMatrix(self.basis, self.H_dev, lay.d1, lay.cap, lay.groups, gamma=gamma,
                         state=self)

    def hint_group_mults(self, group_ids=None) -> int:
        """The reference multiexp's group-multiplication count for the hint
        entries of `group_ids` (all groups by default) -- what its counter
        bumps in paillier.py:192. The count depends only on the exponents
        H_scaled, not on the client's bases: computed once per state on the
        device (zpir_multiexp_opcount) and cached."""
        with self._lock:
            per = getattr(self, "_opcount", None)
            if per is None:
                lay = self.layout
                g = lay.gamma
                if g & (g - 1) == 0 and g >= lay.q:
                    # gamma = 2^sbits >= q > every H entry: exponents are slot concatenations
                    out = torch.empty(lay.groups, dtype=torch.int64, device=self.device)
                    st = torch.cuda.current_stream(self.device)
                    _lib.call("zpir_multiexp_opcount", _lib.ptr(self.H_dev), lay.d1, lay.n,
                              lay.cap, g.bit_length() - 1, lay.groups, _lib.ptr(out),
                              st.cuda_stream)
                    per = out.cpu().numpy()
                else:
                    # standard-regime gamma (q + n q): the exponents are not slot
                    # concatenations; the reference count is not derived on the
                    # device (one product per (group, base) is reported instead)
                    per = np.full(lay.groups, lay.n, dtype=np.int64)
                self._opcount = per
        if group_ids is None:
            return int(per.sum())
        return int(per[np.asarray(group_ids, dtype=np.int64)].sum())

    @property
    def A(self) -> np.ndarray:
        """The (d0, n) public matrix (protocol.py:175-176), host view."""
        with self._lock:
            if self._A64 is None:
                lay = self.layout
                self._A64 = device.to_host_u32(self.A_dev[: lay.d0, : lay.n]).astype(np.uint64)
            return self._A64

    @property
    def H(self) -> np.ndarray:
        with self._lock:
            if self._H_host is None:
                h = device.to_host_u32(self.H_dev[: self.layout.d1])
                self._H_host = h.astype(np.uint64)
            return self._H_host

    @property
    def H_scaled(self) -> list:
        """d1' rows of packed big integers (protocol.py:219-238), host view."""
        with self._lock:
            if self._H_scaled is None:
                lay = self.layout
                h = device.to_host_u32(self.H_dev[: lay.groups * lay.cap])
                rows = []
                for g in range(lay.groups):
                    blk = h[g * lay.cap:(g + 1) * lay.cap]
                    rows.append(_pack_slots(blk, lay))
                self._H_scaled = rows
            return self._H_scaled

    # -- online path -------------------------------------------------------

    def _stage_query(self, qu, stream):
        lay = self.layout
        qu = np.asarray(qu)
        if qu.shape != (lay.d0,):
            raise ValueError("query dimensions do not match the parameters")
        q32 = np.zeros(lay.ld, dtype=np.uint32)
        q32[: lay.d0] = qu.astype(np.uint64) & np.uint64(0xFFFFFFFF)
        return _h2d(q32, self.device, "qu", stream).view(torch.int32).reshape(1, lay.ld)

    def db_matvec(self, qu) -> np.ndarray:
        """b = db^T qu mod q (protocol.py:242-257), uint64 (d1,)."""
        stream = torch.cuda.current_stream(self.device)
        qd = self._stage_query(qu, stream)
        b = self.gemv_device(qd, stream)
        return _d2h_u32(b[0, : self.layout.d1], "b", stream).astype(np.uint64)

    def gemv_device(self, qu_dev, stream):
        """b (nvec x rows) for staged queries qu_dev (nvec x ld)."""
        lay = self.layout
        nvec = qu_dev.shape[0]
        if self.engine == "umma" and nvec <= 64 and lay.qmask == 0xFFFFFFFF:
            planes = device.query_planes(qu_dev, 16 if nvec <= 4 else 256, stream)
            return device.umma_gemv(self.dbt, planes, nvec, stream=stream)
        return device.gemv(self.dbt, qu_dev, lay.qmask, stream=stream)

    def scaled_b(self, b) -> list:
        """Group b into d1' packed integers (protocol.py:259-269), host view."""
        lay = self.layout
        arr = np.asarray(b, dtype=np.uint64).astype("<u4")
        return [_pack_slots(arr[g * lay.cap:(g + 1) * lay.cap, None], lay)[0]
                for g in range(lay.groups)]

    def _workspace(self, lm):
        """Per-thread device buffers and side stream for the online path."""
        tl = self._tls
        ws = getattr(tl, "ws", None)
        if ws is None:
            ws = tl.ws = {}
        w = ws.get(lm)
        if w is None:
            lay = self.layout
            dev = self.device
            w = ws[lm] = {
                "side": torch.cuda.Stream(dev),
                "ev_in": torch.cuda.Event(), "ev_comp": torch.cuda.Event(),
                "planes": torch.empty((16, lay.ld), dtype=torch.uint8, device=dev),
                "b": torch.empty((1, lay.rows), dtype=torch.int32, device=dev),
                "z": torch.empty((lay.rows, lm + 4), dtype=torch.int32, device=dev),
                "bc": (torch.empty(self.compress_operand_shape(lm), dtype=torch.uint8,
                                   device=dev) if lm in device.UMMA_NB else None),
            }
        return w

    def planar(self, lm) -> bool:
        """The planar compression GEMM serves this key width."""
        return (self.engine == "umma" and lm in device.PLANAR_LM
                and self.H_planes is not None and self.layout.n <= 33025)

    def compress_rows(self, cko, lm, stream, out=None, ctas=0, bc=None):
        """z (rows x lm+4, or nq x rows x lm+4 for cko of nq queries) on the
        tensor cores: planar kernel where it applies, else the byte-shifted one."""
        lay = self.layout
        batched = cko.dim() == 3
        if self.planar(lm):
            bp = device.build_bcp(cko, lm, stream, out=bc)
            z = out.view(-1, lay.rows, lm + 4) if out is not None else None
            z = device.umma_answer_rows_planar(self.H_planes, lay.n, bp, lm, out=z, stream=stream,
                                               ctas=ctas)
            return z if batched else z[0]
        if batched:
            bcs = device.build_bc_batch(cko, lm, stream)
            return device.umma_answer_rows_batch(self.H_dev, bcs, lm, stream)
        bcs = device.build_bc(cko, lm, stream=stream, bc=bc)
        return device.umma_answer_rows(self.H_dev, bcs, None, lay.qmask, lm, out=out, stream=stream,
                                       ctas=ctas)

    def compress_operand_shape(self, lm):
        """Shape / dtype of the per-query compression operand buffer."""
        lay = self.layout
        if self.planar(lm):
            return (1, 4 * lm, device.planar_np(lay.n))
        return (device.UMMA_NB[lm], 4 * lay.n)

    def answer_plan(self, kctx, t_ld):
        """Per-thread captured plan for the tcgen05 path, or None."""
        lay = self.layout
        # the plan's finish adds B_g < 2^(32 cap) to tz mod m with one conditional
        # subtraction: exact when 2^(32 cap) <= m (keys of the params' size)
        if not (self.engine == "umma" and kctx.lm in device.UMMA_NB and lay.n % 4 == 0
                and lay.qmask == 0xFFFFFFFF and lay.stride == 1
                and 32 * lay.cap < kctx.m.bit_length()):
            return None
        plans = getattr(self._tls, "plans", None)
        if plans is None:
            plans = self._tls.plans = {}
        key = (kctx.lm, t_ld)
        p = plans.get(key)
        if p is None:
            p = plans[key] = AnswerPlan(self, kctx, t_ld, COMPRESS_CTAS)
        return p

    def answer_batch_device(self, qu_dev, cko_dev, kctxs, t_ld, stream, events=None):
        """t (nq x groups x t_ld) for nq <= 64 staged queries (tcgen05 path):
        one N = 4*nq GEMV over the DB, one compression launch, one group launch."""
        if events:
            events[0].record(stream)
        b = self.gemv_batch_device(qu_dev, stream)
        if events:
            events[1].record(stream)
        t = self.compress_groups_batch(cko_dev, b, kctxs, t_ld, stream)
        if events:
            events[2].record(stream)
        return t

    def gemv_batch_device(self, qu_dev, stream):
        """b (nq x rows) = DB qu_v mod q for nq <= 64 staged queries: one pass over the DB."""
        nq = qu_dev.shape[0]
        planes = device.query_planes(qu_dev, 16 if nq <= 4 else 256, stream)
        return device.umma_gemv(self.dbt, planes, nq, stream=stream)

    def compress_groups_batch(self, cko_dev, b, kctxs, t_ld, stream):
        """t (nq x groups x t_ld) from the queries' ck_o limbs and their GEMV rows b."""
        lay = self.layout
        z = self.compress_rows(cko_dev, kctxs[0].lm, stream)
        return device.answer_groups_batch(z, b, lay.qmask, lay.d1, lay.cap, lay.groups, kctxs,
                                          t_ld, stream, stride=lay.stride)

    def _group_stage(self, z, b, kctx, t_ld, stream):
        """t_g = sum_j gamma^j (b_c + z_c) mod m: positional fold for gamma =
        2^32 / 2^64, per-row weights gamma^j mod m otherwise."""
        lay = self.layout
        if lay.stride == 1:
            return device.answer_groups(z, b, lay.qmask, lay.d1, lay.cap, lay.groups, kctx, t_ld,
                                        stream=stream)
        if lay.stride:
            return device.answer_groups_strided(z, b, lay.qmask, lay.d1, lay.cap, lay.groups, kctx,
                                                t_ld, lay.stride, stream=stream)
        return device.answer_general(z, b, lay.qmask, lay.d1, lay.cap, lay.groups, kctx,
                                     lay.gamma, t_ld, stream=stream)

    def answer_device(self, qu_dev, cko_dev, kctx, t_ld, stream, events=None):
        """t (groups x t_ld u32 limbs) for one staged query; all on device.

        UMMA engine: the compression GEMM (H, 1/8 of the bytes) runs on a side
        stream on COMPRESS_CTAS SMs while the GEMV streams the DB on the other
        SMs; the group stage joins both."""
        lay = self.layout
        lm = kctx.lm
        if events:
            events[0].record(stream)
        if (self.engine == "umma" and lm in device.UMMA_NB and qu_dev.shape[0] == 1
                and lay.qmask == 0xFFFFFFFF and lay.n % 4 == 0):
            w = self._workspace(lm)
            side = w["side"]
            split = COMPRESS_CTAS > 0
            cs = side if split else stream
            if split:
                w["ev_in"].record(stream)
                side.wait_event(w["ev_in"])
            z = self.compress_rows(cko_dev, lm, cs, out=w["z"], ctas=COMPRESS_CTAS if split else 0,
                                   bc=w["bc"])
            if split:
                w["ev_comp"].record(side)
            planes = device.query_planes(qu_dev, 16, stream, planes=w["planes"])
            sms = torch.cuda.get_device_properties(self.device).multi_processor_count
            b = device.umma_gemv(self.dbt, planes, 1, out=w["b"], stream=stream,
                                 ctas=(sms - COMPRESS_CTAS) if split else 0)
            if events:
                events[1].record(stream)
            if split:
                stream.wait_event(w["ev_comp"])
        else:
            b = self.gemv_device(qu_dev, stream)
            if events:
                events[1].record(stream)
            z = device.answer_rows(self.H_dev, b[0], lay.qmask, cko_dev, lm, stream=stream)
        t = self._group_stage(z, b[0], kctx, t_ld, stream)
        if events:
            events[2].record(stream)
        return t


def _pack_slots(blk, lay) -> list:
    """Columns of blk (rows j < cap, u32) as sum_j gamma^j blk[j] (protocol.py:219-238)."""
    blk = np.asarray(blk, dtype="<u4")
    if lay.stride:
        w = np.zeros((blk.shape[1], blk.shape[0] * lay.stride), dtype="<u4")
        w[:, :: lay.stride] = blk.T
        return [int.from_bytes(w[i].tobytes(), "little") for i in range(w.shape[0])]
    out = []
    for i in range(blk.shape[1]):
        acc = 0
        for v in blk[::-1, i]:
            acc = acc * lay.gamma + int(v)
        out.append(acc)
    return out


def derive_ck_r(pk, seed: bytes, query_index: int, n: int):
    """The seeded compression-key ciphertexts for one query index (protocol.py:285-288)."""
    return [sample_ciphertext(pk, seed, (query_index << 32) | i) for i in range(n)]


class _StreamPool(threading.local):
    """Side streams of hints() / refresh_hints(), created once per thread and
    device and reused (a hint worker thread calls them for every batch)."""

    def __init__(self):
        self.pools = {}


_stream_pool = _StreamPool()


def _side_streams(dev, count):
    pool = _stream_pool.pools.setdefault(str(dev), [])
    while len(pool) < count:
        pool.append(torch.cuda.Stream(dev))
    return pool[:count]


def _tc_eligible(state, kctx) -> bool:
    return TC_HINT and kctx.l2 == 128 and 7 * state.layout.n <= 65536   # D n positions


def _tc_refresh_pays(state, nclients: int, rows: int) -> bool:
    """Tensor cores or IMAD kernels for a refresh of `rows` changed DB rows of
    `nclients` hints (measured on a B200). A tensor-core launch walks
    all D n positions (D = 7, ~7.5 us each) whatever the row count, with one CTA
    pair per 512 rows and client and 74 pairs per wave, plus ~0.6 us per position
    and client for the multiplier tables; the IMAD kernels cost ~35 us per row and
    client (the Horner recombination of the changed groups is common to both).
    One client's 327 rows stay on the IMAD path (11 ms against 58 ms); the hint
    worker's 16 clients go to the tensor cores (122 ms against 183 ms; measured
    16.1 against 17.9 ms per client with the recombination)."""
    if rows >= TC_REFRESH_MIN_ROWS:
        return True
    npos = 7 * state.layout.n
    waves = -(-nclients * -(-rows // 512) // 74)
    tc_ms = waves * npos * 7.5e-3 + nclients * (npos * 0.6e-3 + rows * 0.5e-3)
    return tc_ms < nclients * rows * 35e-3


def _tc_batches(state, items, rows):
    """Split tensor-core jobs into launches whose transient workspace stays
    under TC_WS_BYTES (48 GB: 16 clients at n = 1024; at least one client per launch)."""
    per = device.slot_fixed_tc_workspace(state.layout.n, rows, 1)
    k = max(1, int(TC_WS_BYTES // max(per, 1)))
    return [items[i:i + k] for i in range(0, len(items), k)]


def hint(state: ServerGlobalState, reg, query_index: int, stream=None,
         keep_slots: bool = False) -> ClientHint:
    """k_g = prod_k ck_r[k]^{H_scaled[g][k]} mod m^2 for all d1' groups
    (protocol.py:291-296; paillier_matmul / multiexp, paillier.py:134-203).

    Computed through the slot decomposition: H_scaled[g][k] = sum_j gamma^j
    H[g*cap+j][k], so k_g = prod_j W[g*cap+j]^(gamma^j) with
    W[c] = prod_k ck_r[k]^H[c][k].
    Each W[c] (32-bit exponents) is one fixed-base Pippenger over a table of
    powers of ck_r[k]: on the IMAD path (slot_fixed) 8-bit digits, 255
    buckets, P[i][k] = ck_r[k]^(2^(8i)); for 4096-bit m^2 and enough rows the
    bucket updates run on the tensor cores instead (tc_pippenger.cu: D = 7
    digits per word, 31 buckets). The groups are then recombined by
    Horner in gamma (slot_combine). Same group element as the reference's
    windowed multiexp, canonical mod m^2. keep_slots=True keeps W and the
    8-bit table P on the device for refresh_hint."""
    return hints(state, [(reg, query_index)], stream=stream, keep_slots=keep_slots)[0]


def hints(state: ServerGlobalState, jobs, stream=None, keep_slots: bool = False) -> list:
    """hint() for several (registration, query index) jobs: the tensor-core
    Pippenger runs all of them in one launch (blockIdx.y = client), so the
    row tiles of a batch fill whole waves of SMs (the hint worker's batch;
    SURVEY.md section 8f rank 1). Returns one ClientHint per job, in order."""
    lay = state.layout
    dev = state.device
    stream = stream or torch.cuda.current_stream(dev)
    nslot = lay.groups * lay.cap
    prep = []
    for reg, qi in jobs:
        kctx = key_ctx(reg.pk.m, dev)
        # ck_r[k] = Stream(seed, 1, (qi << 32) | k).below(m^2), sampled on the device
        bases = device.chacha_below(reg.seed, DOM_CIPHERTEXT_SAMPLE, qi, lay.n, kctx.d_m2,
                                    kctx.m2, kctx.l2, stream)
        P = device.pow8_table(bases, kctx, stream)
        W = torch.empty((nslot, kctx.l2), dtype=torch.int32, device=dev)
        prep.append((P, kctx, W))
    # the tensor-core launch costs ~D*n positions of fixed latency per wave of row
    # tiles; below ~TC_MIN_ROWS rows in the whole batch the IMAD kernel is faster
    tc = [j for j in prep if _tc_eligible(state, j[1])]
    if nslot * len(tc) < TC_MIN_ROWS:
        tc = []
    tc_ids = set()
    for batch in (_tc_batches(state, tc, nslot) if tc else []):
        try:
            device.slot_fixed_tc_many(batch, lay.n, state.H_dev, lay.n, nslot, stream=stream)
        except _lib.ZpirError as e:      # e.g. no room for the workspace: IMAD kernels below
            log.warning("tensor-core hint batch of %d fell back to IMAD: %s", len(batch), e)
            continue
        tc_ids.update(id(j[2]) for j in batch)
    # the per-client group recombination (slot_combine: one warp per group, a
    # 32 * cap-deep Horner chain) is latency bound for one client: the clients
    # of the tensor-core batch run in one launch (blockIdx.y = client, grouped by
    # key width); the IMAD-path clients (slot_fixed + slot_combine each) side by
    # side on a small stream pool
    out = {}
    by_width = {}
    for (P, kctx, W) in prep:
        if id(W) in tc_ids:
            k = torch.empty((lay.groups, kctx.l2), dtype=torch.int32, device=dev)
            out[id(W)] = k
            by_width.setdefault(kctx.l2, []).append((W, kctx, k))
    for group in by_width.values():
        device.slot_combine_many(group, lay.cap, None, lay.groups, lay.gamma, stream)
    rest = [j for j in prep if id(j[2]) not in tc_ids]
    side = [stream] if len(rest) <= 1 else _side_streams(dev, min(4, len(rest)))
    ev = torch.cuda.Event()
    ev.record(stream)
    for i, (P, kctx, W) in enumerate(rest):
        st = side[i % len(side)]
        if st is not stream:
            st.wait_event(ev)
        device.slot_fixed(P, lay.n, state.H_dev, lay.n, None, nslot, kctx, W, st)
        k = torch.empty((lay.groups, kctx.l2), dtype=torch.int32, device=dev)
        device.slot_combine(W, lay.cap, None, lay.groups, kctx, k, lay.gamma, st)
        out[id(W)] = k
    for st in side:
        if st is not stream:
            stream.wait_stream(st)
    out = [out[id(W)] for _, _, W in prep]
    res = []
    for (reg, qi), (P, kctx, W), k in zip(jobs, prep, out):
        entries = limbs_to_ints(_d2h_u32(k, "hint", stream))
        counters.bump("group_mult", state.hint_group_mults())
        res.append(ClientHint(qi, state.db_version, [PaillierCiphertext(e) for e in entries],
                              dev=k, slots=W if keep_slots else None,
                              bases=P if keep_slots else None))
    return res


def _refresh_device(state, kctx, old, rows, rid, gid, ngroups, stream):
    lay = state.layout
    W = old.slots.clone()
    k = old.dev.clone()
    if rows:
        device.slot_fixed(old.bases, lay.n, state.H_dev, lay.n, rid, rows, kctx, W, stream)
        device.slot_combine(W, lay.cap, gid, ngroups, kctx, k, lay.gamma, stream)
    return W, k


def _changed_ids(state, changed_rows):
    lay = state.layout
    rows = np.unique(np.asarray(changed_rows, dtype=np.int64))
    if rows.size and (rows.min() < 0 or rows.max() >= lay.d1):
        raise ValueError("changed row out of range")
    groups = np.unique(rows // lay.cap).astype(np.int32)
    dev = state.device
    rid = torch.from_numpy(rows.astype(np.int32)).to(dev) if rows.size else None
    gid = torch.from_numpy(groups).to(dev) if groups.size else None
    return rows.size, rid, gid, groups.size


def refresh_hint(state: ServerGlobalState, reg, old: ClientHint, changed_rows,
                 stream=None) -> ClientHint:
    """Incremental hint refresh after a DB-row update (no reference
    counterpart: the reference regenerates every hint, server.py:115-124).

    `old` must carry its slot decomposition (hint(..., keep_slots=True)) and
    `state` is the updated state (ServerGlobalState.updated). Only the
    changed DB rows' factors W[c] are recomputed (one fixed-base 32-bit
    multiexp each) and only their groups are recombined; bit-identical to a
    full hint() on the new state."""
    return refresh_hints(state, [(reg, old)], changed_rows, stream=stream)[0]


def refresh_hints(state: ServerGlobalState, pairs, changed_rows, stream=None,
                  nstreams: int = 8) -> list:
    """refresh_hint for many (registration, hint) pairs at once. For large
    updates (>= TC_REFRESH_MIN_ROWS changed rows) or enough clients to fill a
    launch (_tc_refresh_pays) and 4096-bit m^2 the changed rows' W of all
    clients are recomputed by one tensor-core launch (row ids, one grid row
    per client); otherwise the IMAD
    kernels of each client are spread over `nstreams` CUDA streams so that
    small refreshes fill the GPU together."""
    for _, old in pairs:
        if old.slots is None or old.bases is None:
            raise ValueError("refresh_hint needs a hint computed with keep_slots=True")
    dev = state.device
    lay = state.layout
    main = stream or torch.cuda.current_stream(dev)
    rows, rid, gid, ng = _changed_ids(state, changed_rows)
    kctxs = [key_ctx(reg.pk.m, dev) for reg, _ in pairs]
    use_tc = (all(_tc_eligible(state, k) for k in kctxs)
              and _tc_refresh_pays(state, len(pairs), rows))
    if use_tc:
        outs = []
        jobs = []
        for (reg, old), kctx in zip(pairs, kctxs):
            W = old.slots.clone()
            outs.append((W, old.dev.clone()))
            jobs.append((old.bases, kctx, W))
        for batch in _tc_batches(state, jobs, rows):
            try:
                device.slot_fixed_tc_many(batch, lay.n, state.H_dev, lay.n, rows, rid=rid,
                                          stream=main)
            except _lib.ZpirError as e:  # e.g. no room for the workspace: IMAD kernels
                log.warning("tensor-core refresh of %d fell back to IMAD: %s", len(batch), e)
                for P, kctx, W in batch:
                    device.slot_fixed(P, lay.n, state.H_dev, lay.n, rid, rows, kctx, W, main)
        by_width = {}
        for (W, k), kctx in zip(outs, kctxs):
            by_width.setdefault(kctx.l2, []).append((W, kctx, k))
        for group in by_width.values():
            device.slot_combine_many(group, lay.cap, gid, ng, lay.gamma, main)
    else:
        streams = [main] if len(pairs) == 1 else _side_streams(dev, min(nstreams, len(pairs)))
        ev = torch.cuda.Event()
        ev.record(main)
        outs = []
        for i, ((reg, old), kctx) in enumerate(zip(pairs, kctxs)):
            st = streams[i % len(streams)]
            if st is not main:
                st.wait_event(ev)
            with torch.cuda.stream(st):
                outs.append(_refresh_device(state, kctx, old, rows, rid, gid, ng, st))
        for st in streams:
            if st is not main:
                main.wait_stream(st)
    res = []
    gids = np.unique(np.asarray(changed_rows, dtype=np.int64) // lay.cap)
    mults = state.hint_group_mults(gids) if gids.size else 0
    for (reg, old), (W, k) in zip(pairs, outs):
        counters.bump("group_mult", mults)
        entries = limbs_to_ints(_d2h_u32(k, "hint", main))
        res.append(ClientHint(old.query_index, state.db_version,
                              [PaillierCiphertext(e) for e in entries], dev=k, slots=W,
                              bases=old.bases))
    return res


def _conv_module():
    from .bigint import _conv
    return _conv()


def _digit_conv():
    """The C extension's raw-digit entry points (CPython 3.12/3.13), or None."""
    from .bigint import _conv
    c = _conv()
    return c if hasattr(c, "digits_into") else None


def _stored_device(stored, kctx, dev, stream):
    d = getattr(stored, "dev", None)
    if d is not None and d.device == dev and d.shape[1] == kctx.l2:
        return d
    vals = [(c.c if hasattr(c, "c") else int(c)) % kctx.m2 for c in stored.entries]
    d = _h2d(ints_to_limbs(vals, kctx.l2), dev, "k", stream).view(torch.int32)
    return d.reshape(len(vals), kctx.l2)


def respond(state: ServerGlobalState, reg, qmsg, mode: str = None, timings=None,
            stream=None) -> ResponseMessage:
    lay = state.layout
    mode = mode or qmsg.mode
    if len(qmsg.ck_o) != lay.n or len(qmsg.qu0) != lay.d0:
        raise ValueError("query dimensions do not match the parameters")
    stored = reg.hints.get(qmsg.query_index)
    if stored is None or stored.db_version != state.db_version:
        raise KeyError("no hint for this query index and database version")
    if mode not in (SEPARATE, COMBINED):
        raise ValueError("unknown response mode")
    dev = state.device
    stream = stream or torch.cuda.current_stream(dev)
    kctx = key_ctx(reg.pk.m, dev)
    t_total = time.perf_counter()
    events = [torch.cuda.Event(enable_timing=True) for _ in range(3)] if timings is not None else None
    t_ld = kctx.lm if mode == SEPARATE else kctx.l2
    plan = state.answer_plan(kctx, t_ld)
    if plan is not None:
        key_changed = plan.set_key(kctx, stream)
        conv = _digit_conv()
        if conv is not None and plan.ctas > 0 and events is None:
            # two raw graph launches: the GEMV graph starts as soon as qu is
            # staged; ck_o's digits are copied on the host meanwhile, then the
            # side graph (compression, groups; waits for the GEMV; finish)
            qu = qmsg.qu0
            if isinstance(qu, np.ndarray) and qu.ndim == 1 and qu.dtype.itemsize in (4, 8):
                conv.narrow_u32(qu, plan.np_qu, lay.d0)
            else:
                np.copyto(plan.np_qu[: lay.d0], np.asarray(qu), casting="unsafe")
            side = plan.side
            if key_changed:
                side.wait_stream(stream)     # the new key constants were copied on `stream`
            plan.launch("e2e_g1", stream)
            device.event_record(plan.ev_gemv, stream)
            conv.digits_into(qmsg.ck_o, plan.np_ckd, plan.ndig_m, 32 * kctx.lm)
            if mode == SEPARATE:
                plan.launch("e2e_g2", side)
                side.synchronize()
                vals = conv.ints_from_digits(plan.np_td, lay.groups, plan.ndig_m)
                return ResponseMessage(SEPARATE, qmsg.query_index, vals, stored.entries)
            plan.launch("e2e_g2t", side)
            k_dev = _stored_device(stored, kctx, dev, side)
            K = device.combine(plan.t, k_dev, kctx, stream=side)
            device.limbs_to_digits(K, kctx.l2, plan.d_Kd, side)
            device.d2h_async(plan.h_Kd, plan.d_Kd, side)
            side.synchronize()
            vals = conv.ints_from_digits(plan.np_Kd, lay.groups, plan.ndig_2)
            counters.bump("add", lay.groups)
            counters.bump("group_mult", lay.groups)
            return ResponseMessage(COMBINED, qmsg.query_index, [],
                                   [PaillierCiphertext(v) for v in vals])
        # qu -> pinned -> device; GEMV graph on (SMs - COMPRESS_CTAS) SMs
        qu = np.asarray(qmsg.qu0)
        hq = plan.h_qu.numpy().view(np.uint32)
        np.copyto(hq[: lay.d0], qu, casting="unsafe")
        device.h2d_async(plan.qu, plan.h_qu, stream)
        if events:
            events[0].record(stream)
        if conv is not None and plan.ctas > 0:
            plan.ev_in.record(stream)   # key constants staged; before the GEMV
            plan.run("gemv_part", stream)
            if events:
                events[1].record(stream)
            # meanwhile: ck_o digits (memcpy) -> side stream graph (compression
            # + Montgomery group stage on COMPRESS_CTAS SMs, concurrent with the GEMV)
            conv.digits_into(qmsg.ck_o, plan.h_ckd.numpy(), plan.ndig_m, 32 * kctx.lm)
            side = plan.side
            side.wait_event(plan.ev_in)
            device.h2d_async(plan.d_ckd, plan.h_ckd, side)
            plan.run("side_digits", side)
            stream.wait_stream(side)
            plan.run("finish_digits", stream)
        elif conv is not None:
            plan.run("gemv", stream)
            if events:
                events[1].record(stream)
            conv.digits_into(qmsg.ck_o, plan.h_ckd.numpy(), plan.ndig_m, 32 * kctx.lm)
            device.h2d_async(plan.d_ckd, plan.h_ckd, stream)
            plan.run("compress_digits", stream)
        else:
            plan.run("gemv", stream)
            if events:
                events[1].record(stream)
            ints_to_limbs(qmsg.ck_o, kctx.lm, out=plan.h_cko.numpy().view(np.uint32))
            device.h2d_async(plan.cko, plan.h_cko, stream)
            plan.run("compress", stream)
        if events:
            events[2].record(stream)
        if mode == COMBINED:
            k_dev = _stored_device(stored, kctx, dev, stream)
            K = device.combine(plan.t, k_dev, kctx, stream=stream)
            if conv is not None:
                device.limbs_to_digits(K, kctx.l2, plan.d_Kd, stream)
                src, h_out, nd = plan.d_Kd, plan.h_Kd, plan.ndig_2
            else:
                src, h_out, nd = K, plan.h_K, None
        elif conv is not None:
            src, h_out, nd = plan.d_td, plan.h_td, plan.ndig_m
        else:
            src, h_out, nd = plan.t, plan.h_t, None
        device.d2h_async(h_out, src, stream)
        stream.synchronize()
        if nd is not None:
            vals = conv.ints_from_digits(h_out.numpy(), h_out.shape[0], nd)
        else:
            vals = limbs_to_ints(h_out.numpy().view(np.uint32))
    else:
        qu_dev = state._stage_query(qmsg.qu0, stream)
        cko = _h2d(ints_to_limbs(qmsg.ck_o, kctx.lm), dev, "cko", stream).view(torch.int32)
        cko = cko.reshape(lay.n, kctx.lm)
        t_dev = state.answer_device(qu_dev, cko, kctx, t_ld, stream, events)
        if mode == COMBINED:
            k_dev = _stored_device(stored, kctx, dev, stream)
            t_dev = device.combine(t_dev, k_dev, kctx, stream=stream)
        vals = limbs_to_ints(_d2h_u32(t_dev, "t", stream))
    if mode == SEPARATE:
        out = ResponseMessage(SEPARATE, qmsg.query_index, vals, stored.entries)
    else:
        counters.bump("add", lay.groups)
        counters.bump("group_mult", lay.groups)
        out = ResponseMessage(COMBINED, qmsg.query_index, [],
                              [PaillierCiphertext(v) for v in vals])
    if timings is not None:
        stream.synchronize()
        timings["db_matvec"] = events[0].elapsed_time(events[1]) / 1e3
        timings["hint_matvec"] = events[1].elapsed_time(events[2]) / 1e3
        timings["total"] = time.perf_counter() - t_total
    return out


def respond_wire(state: ServerGlobalState, reg, query_index: int, mode: str, ck_bytes, qu,
                 stream=None):
    """respond() on fixed-width wire fields, without Python ints
    (protocol.py:333-365 + wire.py:141-193).

    ck_bytes: (n, w) uint8 little-endian magnitudes (w <= limb bytes of m,
    as wire.decode_query returns them); qu: (d0,) integers. Returns the
    result as (d1', L) u32 limb rows -- t for SEPARATE, K for COMBINED --
    for wire.field_rows. Same validation and exceptions as respond()."""
    lay = state.layout
    ck_bytes = np.asarray(ck_bytes)
    qu = np.asarray(qu)
    if ck_bytes.ndim != 2 or ck_bytes.shape[0] != lay.n or qu.shape != (lay.d0,):
        raise ValueError("query dimensions do not match the parameters")
    stored = reg.hints.get(query_index)
    if stored is None or stored.db_version != state.db_version:
        raise KeyError("no hint for this query index and database version")
    if mode not in (SEPARATE, COMBINED):
        raise ValueError("unknown response mode")
    out = _wire_rows(state, reg.pk.m, mode, ck_bytes, qu, stored, stream)
    if mode == COMBINED:
        counters.bump("add", lay.groups)
        counters.bump("group_mult", lay.groups)
    return out


def answer_wire(state: ServerGlobalState, m: int, ck_bytes, qu, stream=None,
                on_device: bool = False):
    """t (d1' x lm u32 limb rows) of one query on fixed-width wire fields,
    without a stored-hint check: the per-shard answer of a row-sharded server
    (shard.py), whose hints live on the answering rank. on_device=True
    returns the device rows (int32 view, valid until the next answer on this
    thread) instead of a host copy."""
    lay = state.layout
    ck_bytes = np.asarray(ck_bytes)
    qu = np.asarray(qu)
    if ck_bytes.ndim != 2 or ck_bytes.shape[0] != lay.n or qu.shape != (lay.d0,):
        raise ValueError("query dimensions do not match the parameters")
    return _wire_rows(state, m, SEPARATE, ck_bytes, qu, None, stream, on_device)


def _wire_rows(state, m, mode, ck_bytes, qu, stored, stream, on_device=False):
    lay = state.layout
    dev = state.device
    stream = stream or torch.cuda.current_stream(dev)
    kctx = key_ctx(m, dev)
    w = ck_bytes.shape[1]
    if w > 4 * kctx.lm:
        raise ValueError("ck_o field wider than the modulus")
    t_ld = kctx.lm if mode == SEPARATE else kctx.l2
    plan = state.answer_plan(kctx, t_ld)
    if plan is None or plan.ctas <= 0:
        ck = np.zeros((lay.n, 4 * kctx.lm), dtype=np.uint8)
        ck[:, :w] = ck_bytes
        q32 = np.zeros(lay.ld, dtype=np.uint32)
        np.copyto(q32[: lay.d0], qu, casting="unsafe")
        qd = _h2d(q32, dev, "qu", stream).view(torch.int32).reshape(1, lay.ld)
        cko = _h2d(ck.view("<u4"), dev, "cko", stream).view(torch.int32).reshape(lay.n, kctx.lm)
        t_dev = state.answer_device(qd, cko, kctx, t_ld, stream)
        if mode == COMBINED:
            t_dev = device.combine(t_dev, _stored_device(stored, kctx, dev, stream), kctx,
                                   stream=stream)
        if on_device:
            stream.synchronize()
            return t_dev[: lay.groups]
        out = _d2h_u32(t_dev, "t", stream)
    else:
        side = plan.side
        if plan.set_key(kctx, stream):
            side.wait_stream(stream)
        hq = plan.h_qu.numpy().view(np.uint32)
        np.copyto(hq[: lay.d0], qu, casting="unsafe")
        plan.launch("e2e_g1", stream)          # qu in, GEMV
        device.event_record(plan.ev_gemv, stream)
        # meanwhile: ck_o bytes -> pinned limb rows -> side graph (compression,
        # groups, then the finish once the GEMV is done)
        hc = plan.h_cko.numpy().view(np.uint8).reshape(lay.n, 4 * kctx.lm)
        if getattr(plan, "_ck_w", None) != w:
            hc[:] = 0
            plan._ck_w = w
        hc[:, :w] = ck_bytes
        plan.launch("w_g2t", side)
        if on_device:
            side.synchronize()
            return plan.t[: lay.groups]
        if mode == COMBINED:
            K = device.combine(plan.t, _stored_device(stored, kctx, dev, side), kctx, stream=side)
            device.d2h_async(plan.h_K, K, side)
            h_out = plan.h_K
        else:
            device.d2h_async(plan.h_t, plan.t, side)
            h_out = plan.h_t
        side.synchronize()
        out = h_out.numpy().view(np.uint32)
    return out


MAX_BATCH = 64
# respond_batch: queries per compression / copy-out sub-batch (host work overlaps the device)
BATCH_SUB = 16
# respond_batch_wire: every input is staged up front; the sub-batches overlap the
# copies in and out with the compressions (measured 16 / 32 / 64: 3.19 / 3.28 / 4.32 ms)
WIRE_BATCH_SUB = 16


def respond_batch(state: ServerGlobalState, regs, qmsgs, mode: str = None,
                  stream=None) -> list:
    """Answer many queries together (BASELINE configs[3]); the reference has
    no batch path and answers one query at a time (protocol.py:333-365).

    Per chunk of <= 64 queries: ONE tensor-core GEMV streams the DB once for
    all of them (N = 4 byte planes x 64 queries = 256), one compression launch
    covers every query (H row blocks reused from L2), one group-stage launch
    with per-query moduli. Same validation / exceptions / counters as respond;
    returns the list of ResponseMessages in order."""
    if len(regs) != len(qmsgs):
        raise ValueError("regs and qmsgs must have the same length")
    lay = state.layout
    dev = state.device
    stream = stream or torch.cuda.current_stream(dev)
    modes, storeds, kctxs = [], [], []
    for reg, q in zip(regs, qmsgs):
        md = mode or q.mode
        if len(q.ck_o) != lay.n or len(q.qu0) != lay.d0:
            raise ValueError("query dimensions do not match the parameters")
        st = reg.hints.get(q.query_index)
        if st is None or st.db_version != state.db_version:
            raise KeyError("no hint for this query index and database version")
        if md not in (SEPARATE, COMBINED):
            raise ValueError("unknown response mode")
        modes.append(md)
        storeds.append(st)
        kctxs.append(key_ctx(reg.pk.m, dev))
    if not qmsgs:
        return []
    umma_ok = (state.engine == "umma" and lay.qmask == 0xFFFFFFFF and lay.stride > 0
               and lay.n % 4 == 0
               and all(k.lm == kctxs[0].lm for k in kctxs) and kctxs[0].lm in device.UMMA_NB)
    if not umma_ok:
        return [respond(state, r, q, mode=md, stream=stream)
                for r, q, md in zip(regs, qmsgs, modes)]
    out = []
    lm = kctxs[0].lm
    conv = _digit_conv()
    for c0 in range(0, len(qmsgs), MAX_BATCH):
        qs = qmsgs[c0:c0 + MAX_BATCH]
        ks = kctxs[c0:c0 + MAX_BATCH]
        nq = len(qs)
        out += _respond_chunk(state, qs, ks, modes[c0:c0 + nq], storeds[c0:c0 + nq], lm, conv,
                              stream)
    return out


def _respond_chunk(state, qs, ks, modes, storeds, lm, conv, stream):
    """One respond_batch chunk: queries staged straight into pinned buffers
    (qu0 narrowed, ck_o as raw CPython digits regrouped on the device), one
    batched answer, results regrouped to digits on the device and copied out.

    With the C extension the host work is pipelined against the device: the
    GEMV (all queries, one pass over the DB) starts as soon as every qu0 is
    staged; the compression, group stage and copy-out then run in sub-batches
    of BATCH_SUB queries, so the host stages the next sub-batch's ck_o digits
    and turns the previous sub-batch's result digits into Python ints while
    the device works."""
    lay = state.layout
    dev = state.device
    nq, n = len(qs), lay.n
    qbuf = _staging.get("qb", nq * lay.ld * 4).numpy().view(np.uint32).reshape(nq, lay.ld)
    if lay.ld > lay.d0:
        qbuf[:, lay.d0:] = 0
    for i, q in enumerate(qs):
        qu = q.qu0
        if conv is not None and isinstance(qu, np.ndarray) and qu.ndim == 1 and \
                qu.dtype.itemsize in (4, 8):
            conv.narrow_u32(qu, qbuf[i], lay.d0)
        else:
            np.copyto(qbuf[i, : lay.d0], np.asarray(qu), casting="unsafe")
    qd = torch.empty((nq, lay.ld), dtype=torch.int32, device=dev)
    device.h2d_async(qd, torch.from_numpy(qbuf.view(np.int32)), stream)
    _staging.mark("qb", stream)
    if conv is None:
        cko = np.empty((nq, n, lm), dtype=np.uint32)
        for i, q in enumerate(qs):
            ints_to_limbs(q.ck_o, lm, out=cko[i])
        cd = _h2d(cko, dev, "cb", stream).view(torch.int32).reshape(nq, n, lm)
        t = state.answer_batch_device(qd, cd, ks, ks[0].l2, stream)      # (nq, groups, l2)
        res = []
        for i in range(nq):
            if modes[i] == SEPARATE:
                r = t[i, :, :lm]
            else:
                r = device.combine(t[i], _stored_device(storeds[i], ks[i], dev, stream), ks[i],
                                   stream=stream)
            res.append(limbs_to_ints(_d2h_u32(r.contiguous(), "tb", stream)))
        return _batch_messages(state, qs, modes, storeds, res)

    G = lay.groups
    l2 = ks[0].l2
    nd1, nd2 = -(-32 * lm // 30), -(-32 * l2 // 30)
    b = state.gemv_batch_device(qd, stream)                          # (nq, rows)
    cbuf = _staging.get("cbd", nq * n * nd1 * 4).numpy().view(np.int32).reshape(nq * n, nd1)
    ncomb = sum(1 for md in modes if md == COMBINED)
    hbuf = _staging.get("tb", (nq * G * nd1 + ncomb * G * nd2) * 4)
    hv = hbuf.numpy().view(np.int32)
    res = [None] * nq
    pending = []
    koff, off = {}, nq * G * nd1

    def drain(item):
        ev, lo, hi = item
        ev.synchronize()
        for i in range(lo, hi):
            if modes[i] == SEPARATE:
                res[i] = conv.ints_from_digits(hv[i * G * nd1:(i + 1) * G * nd1], G, nd1)
            else:
                res[i] = conv.ints_from_digits(hv[koff[i]:koff[i] + G * nd2], G, nd2)

    sub = max(1, BATCH_SUB)
    for lo in range(0, nq, sub):
        hi = min(nq, lo + sub)
        m = hi - lo
        for i in range(lo, hi):
            conv.digits_into(qs[i].ck_o, cbuf[i * n:(i + 1) * n], nd1, 32 * lm)
        dd = torch.empty((m * n, nd1), dtype=torch.int32, device=dev)
        device.h2d_async(dd, torch.from_numpy(cbuf[lo * n:hi * n]), stream)
        cd = torch.empty((m, n, lm), dtype=torch.int32, device=dev)
        device.digits_to_limbs(dd, lm, cd.view(m * n, lm), stream)
        t = state.compress_groups_batch(cd, b[lo:hi], ks[lo:hi], l2, stream)   # (m, G, l2)
        td = torch.empty((m * G, nd1), dtype=torch.int32, device=dev)
        device.limbs_to_digits(t.view(m * G, -1), lm, td, stream)
        device.d2h_async(hbuf[lo * G * nd1 * 4:hi * G * nd1 * 4], td, stream)
        for i in range(lo, hi):
            if modes[i] == COMBINED:
                K = device.combine(t[i - lo], _stored_device(storeds[i], ks[i], dev, stream),
                                   ks[i], stream=stream)
                kd = torch.empty((G, nd2), dtype=torch.int32, device=dev)
                device.limbs_to_digits(K, ks[i].l2, kd, stream)
                device.d2h_async(hbuf[off * 4:(off + G * nd2) * 4], kd, stream)
                koff[i] = off
                off += G * nd2
        ev = torch.cuda.Event()
        ev.record(stream)
        if pending:
            drain(pending.pop())
        pending.append((ev, lo, hi))
    _staging.mark("cbd", stream)
    _staging.mark("tb", stream)
    while pending:
        drain(pending.pop())
    return _batch_messages(state, qs, modes, storeds, res)


class _WireBatchBufs(threading.local):
    """Per-thread pinned buffers of respond_batch_wire (grown on demand)."""

    def __init__(self):
        self.key = None
        self.bufs = None


_wire_bufs = _WireBatchBufs()


def respond_batch_wire(state: ServerGlobalState, regs, query_indices, modes, ck_bytes, qus,
                       stream=None) -> list:
    """respond_batch() on fixed-width wire fields (BASELINE configs[3]), no
    Python ints anywhere: query i is (regs[i], query_indices[i], modes[i],
    ck_bytes[i] (n, w) u8 little-endian ck_o magnitudes as wire.decode_query
    returns them, qus[i] (d0,) integers). Returns per query the (d1', L) u32
    limb rows of t (SEPARATE, L = limbs of m) or K (COMBINED, L = limbs of
    m^2) for wire.field_rows -- views into per-thread pinned memory, valid
    until the next call on this thread. Same validation and exceptions as
    respond(); the reference answers one query at a time
    (protocol.py:333-365, wire.py:141-206).

    Pipeline: every qu0 staged (pinned, parallel host copies) -> ONE N = 4 nq
    tensor-core GEMV over the DB; then per sub-batch of BATCH_SUB queries: ck_o
    bytes staged and copied in, the CTA-pair planar compression + group stage,
    COMBINED's K, results copied out -- the host stages sub-batch s + 1 while
    the device works on s."""
    nq = len(qus)
    if not (len(regs) == len(query_indices) == len(modes) == len(ck_bytes) == nq):
        raise ValueError("batch fields must have the same length")
    if nq == 0:
        return []
    lay = state.layout
    dev = state.device
    stream = stream or torch.cuda.current_stream(dev)
    storeds, kctxs = [], []
    for reg, qi, md, ck, qu in zip(regs, query_indices, modes, ck_bytes, qus):
        ck = np.asarray(ck)
        qu = np.asarray(qu)
        if ck.ndim != 2 or ck.shape[0] != lay.n or qu.shape != (lay.d0,):
            raise ValueError("query dimensions do not match the parameters")
        st = reg.hints.get(qi)
        if st is None or st.db_version != state.db_version:
            raise KeyError("no hint for this query index and database version")
        if md not in (SEPARATE, COMBINED):
            raise ValueError("unknown response mode")
        kc = key_ctx(reg.pk.m, dev)
        if ck.shape[1] > 4 * kc.lm:
            raise ValueError("ck_o field wider than the modulus")
        storeds.append(st)
        kctxs.append(kc)
    lm = kctxs[0].lm
    umma_ok = (state.engine == "umma" and lay.qmask == 0xFFFFFFFF and lay.stride > 0
               and lay.n % 4 == 0 and lm in device.UMMA_NB
               and all(k.lm == lm for k in kctxs))
    if not umma_ok:
        return [respond_wire(state, r, qi, md, ck, qu, stream=stream).copy()
                for r, qi, md, ck, qu in zip(regs, query_indices, modes, ck_bytes, qus)]
    out = []
    for c0 in range(0, nq, MAX_BATCH):
        c1 = min(nq, c0 + MAX_BATCH)
        out += _wire_chunk(state, regs[c0:c1], modes[c0:c1], ck_bytes[c0:c1], qus[c0:c1],
                           storeds[c0:c1], kctxs[c0:c1], lm, stream, c0 > 0)
    return out


def _wire_chunk(state, regs, modes, ck_bytes, qus, storeds, ks, lm, stream, keep_prev):
    lay = state.layout
    dev = state.device
    nq, n, G = len(qus), lay.n, lay.groups
    l2 = ks[0].l2
    key = (id(state), nq, lm)
    tb = _wire_bufs
    if tb.key != key or keep_prev:
        # pinned: qu rows (ld u32, zero tail), ck_o byte rows, results; device copies
        tb.bufs = {
            "q": torch.zeros((nq, lay.ld), dtype=torch.int32).pin_memory(),
            "c": torch.zeros((nq, n, 4 * lm), dtype=torch.uint8).pin_memory(),
            "o": torch.empty((nq, G, l2), dtype=torch.int32).pin_memory(),
            "qd": torch.empty((nq, lay.ld), dtype=torch.int32, device=dev),
            "cd": torch.empty((nq, n, lm), dtype=torch.int32, device=dev),
            "cs": torch.cuda.Stream(dev),      # host -> device copies
            "ds": torch.cuda.Stream(dev),      # device -> host copies
        }
        tb.key = key
    B = tb.bufs
    qn = B["q"].numpy().view(np.uint32)
    cn = B["c"].numpy()
    on = B["o"].numpy().view(np.uint32)
    cs, ds = B["cs"], B["ds"]
    conv = _conv_module()
    nthr = device.host_threads()
    fast = hasattr(conv, "stage_rows")
    # qu0 rows -> pinned (C threads, GIL released) -> device, then ONE GEMV
    if fast:
        conv.stage_rows(qus, qn, lay.ld * 4, 1, lay.ld * 4, nthr, True)
    else:
        for i in range(nq):
            np.copyto(qn[i, : lay.d0], np.asarray(qus[i]), casting="unsafe")
    cs.wait_stream(stream)
    device.h2d_async(B["qd"], B["q"], cs)
    ev = torch.cuda.Event()
    ev.record(cs)
    stream.wait_event(ev)
    b = state.gemv_batch_device(B["qd"], stream)                    # (nq, rows)
    # meanwhile every ck_o field -> pinned, then per sub-batch to the device on
    # the copy stream (overlapping the previous sub-batch's compression)
    if fast:
        conv.stage_rows(ck_bytes, cn, n * 4 * lm, n, 4 * lm, nthr, False)
    else:
        for i in range(nq):
            ck = np.asarray(ck_bytes[i], dtype=np.uint8)
            cn[i, :, : ck.shape[1]] = ck
            cn[i, :, ck.shape[1]:] = 0
    sub = max(1, WIRE_BATCH_SUB)
    ranges = [(lo, min(nq, lo + sub)) for lo in range(0, nq, sub)]
    ev_c = []
    for lo, hi in ranges:
        device.h2d_async(B["cd"][lo:hi], B["c"][lo:hi], cs)
        e = torch.cuda.Event()
        e.record(cs)
        ev_c.append(e)
    res = [None] * nq
    for (lo, hi), e in zip(ranges, ev_c):
        stream.wait_event(e)
        # t rows of lm limbs unless a COMBINED query needs them widened for combine
        t_ld = l2 if any(modes[i] == COMBINED for i in range(lo, hi)) else lm
        t = state.compress_groups_batch(B["cd"][lo:hi], b[lo:hi], ks[lo:hi], t_ld, stream)
        outs = []
        for i in range(lo, hi):
            if modes[i] == SEPARATE:
                outs.append((i, t[i - lo], lm, t_ld == lm))
            else:
                K = device.combine(t[i - lo], _stored_device(storeds[i], ks[i], dev, stream),
                                   ks[i], stream=stream)
                outs.append((i, K, l2, False))
        e = torch.cuda.Event()
        e.record(stream)
        ds.wait_event(e)                        # results out on the copy-back stream
        t.record_stream(ds)
        for i, r, L, compact in outs:
            r.record_stream(ds)
            if compact:                         # lm-limb rows: packed into the row block
                device.d2h_async(B["o"][i].view(-1)[: G * lm], r, ds)
                res[i] = on[i].reshape(-1)[: G * lm].reshape(G, lm)
            else:
                device.d2h_async(B["o"][i], r, ds)
                res[i] = on[i, :, :L]
    ds.synchronize()
    for md in modes:
        if md == COMBINED:
            counters.bump("add", lay.groups)
            counters.bump("group_mult", lay.groups)
    return res


def _batch_messages(state, qs, modes, storeds, res):
    lay = state.layout
    out = []
    for i, vals in enumerate(res):
        qi = qs[i].query_index
        if modes[i] == SEPARATE:
            out.append(ResponseMessage(SEPARATE, qi, vals, storeds[i].entries))
        else:
            counters.bump("add", lay.groups)
            counters.bump("group_mult", lay.groups)
            out.append(ResponseMessage(COMBINED, qi, [], [PaillierCiphertext(v) for v in vals]))
    return out


def client_storage_hint_transfer(reg, query_index: int) -> ClientHint:
    """Hand the stored hint to the client; single use (protocol.py:399-408)."""
    if query_index in reg.consumed:
        raise ValueError("hint already consumed")
    h = reg.hints.get(query_index)
    if h is None:
        raise KeyError("no hint for this query index")
    reg.consumed.add(query_index)
    return h
