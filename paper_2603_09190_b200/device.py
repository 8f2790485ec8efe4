"""Device selection, pinned staging and thin wrappers over the C ABI.

Every function here takes/returns torch tensors on a CUDA device and calls
one extern "C" entry point on the caller's current stream. torch is used for
device memory, streams and events only.
"""

import ctypes
import threading

import numpy as np
import torch

from . import _lib


def require_cuda(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise RuntimeError("paper_2603_09190_b200 needs a CUDA device (B200, sm_100a); "
                           "there is no CPU fallback")
    _lib.load()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device(device)


def u32_tensor(arr, device) -> torch.Tensor:
    """Host uint32 array -> device int32 tensor holding the same bits."""
    a = np.ascontiguousarray(arr, dtype=np.uint32)
    return torch.from_numpy(a.view(np.int32)).to(device, non_blocking=False)


def to_host_u32(t: torch.Tensor) -> np.ndarray:
    return t.cpu().numpy().view(np.uint32)


def _s(stream):
    return _lib.stream_handle(stream)


def transpose_db(db_dev, d0, d1, rows, ld, stream=None):
    out = torch.empty((rows, ld), dtype=torch.uint8, device=db_dev.device)
    _lib.call("zpir_transpose_db", _lib.ptr(db_dev), d0, d1, d1, _lib.ptr(out), rows, ld, _s(stream))
    return out


def global_hint(dbt, A_dev, n, qmask, stream=None):
    rows, ld = dbt.shape
    H = torch.empty((rows, n), dtype=torch.int32, device=dbt.device)
    _lib.call("zpir_global_hint", _lib.ptr(dbt), rows, ld, _lib.ptr(A_dev), A_dev.shape[1], n,
              _lib.ptr(H), qmask, _s(stream))
    return H


def gemv(dbt, qu_dev, qmask, out=None, ws=None, stream=None):
    """b = DB * qu mod 2^32 for qu of shape (nvec, ld) (int32 bits)."""
    rows, ld = dbt.shape
    nvec = qu_dev.shape[0]
    if out is None:
        out = torch.empty((nvec, rows), dtype=torch.int32, device=dbt.device)
    if ws is None:
        ws = torch.empty(int(_lib.lib().zpir_gemv_workspace_bytes(ld, nvec)) // 4,
                         dtype=torch.int32, device=dbt.device)
    _lib.call("zpir_gemv", _lib.ptr(dbt), rows, ld, _lib.ptr(qu_dev), nvec, _lib.ptr(out), qmask,
              _lib.ptr(ws), _s(stream))
    return out


def answer_rows(H, b, qmask, cko, lm, out=None, stream=None):
    rows, n = H.shape
    if out is None:
        out = torch.empty((rows, lm + 4), dtype=torch.int32, device=H.device)
    _lib.call("zpir_answer_rows", _lib.ptr(H), rows, n, _lib.ptr(b), qmask, _lib.ptr(cko), lm,
              _lib.ptr(out), _s(stream))
    return out


def answer_groups(z, b, qmask, d1, cap, groups, kctx, t_ld, out=None, stream=None):
    lm = kctx.lm
    nchunks = max(2, -(-(cap + lm + 4) // lm))
    rpow = kctx.d_rpow(nchunks)
    fast0 = 1 if kctx.cm.R < 2 * kctx.m else 0
    if out is None:
        out = torch.empty((groups, t_ld), dtype=torch.int32, device=z.device)
    _lib.call("zpir_answer_groups", _lib.ptr(z), _lib.ptr(b), qmask, d1, cap, groups, lm,
              _lib.ptr(kctx.d_m), kctx.cm.np, _lib.ptr(rpow), nchunks, fast0, _lib.ptr(out), t_ld,
              _s(stream))
    return out


def combine(t, k, kctx, out=None, stream=None):
    groups = t.shape[0]
    if out is None:
        out = torch.empty((groups, kctx.l2), dtype=torch.int32, device=t.device)
    _lib.call("zpir_combine", _lib.ptr(t), _lib.ptr(k), groups, kctx.l2, _lib.ptr(kctx.d_m2),
              kctx.c2.np, _lib.ptr(kctx.d_r2sq), _lib.ptr(kctx.d_mr), _lib.ptr(out), _s(stream))
    return out


def mulmod(a, b, limbs, d_n, np_, d_r2, stream=None):
    count = a.shape[0]
    out = torch.empty_like(a)
    _lib.call("zpir_mulmod", _lib.ptr(a), _lib.ptr(b), count, limbs, _lib.ptr(d_n), np_,
              _lib.ptr(d_r2), _lib.ptr(out), _s(stream))
    return out


def multiexp(bases, E, rows, rs, bs, ls, elimbs, kctx, stream=None):
    """rows x (prod_k bases[k]^e(g,k) mod m^2); bases (n, l2) canonical."""
    n = bases.shape[0]
    l2 = kctx.l2
    ws_bytes = int(_lib.lib().zpir_multiexp_workspace_bytes(n, rows, elimbs, l2))
    ws = torch.empty(ws_bytes // 4 + 64, dtype=torch.int32, device=bases.device)
    out = torch.empty((rows, l2), dtype=torch.int32, device=bases.device)
    _lib.call("zpir_multiexp", _lib.ptr(bases), n, _lib.ptr(E), rows, rs, bs, ls, elimbs, l2,
              _lib.ptr(kctx.d_m2), kctx.c2.np, _lib.ptr(kctx.d_r2sq), _lib.ptr(out),
              _lib.ptr(ws), ws_bytes, _s(stream))
    return out


# ---- tcgen05 (UMMA) engine ----------------------------------------------------

UMMA_NB = {32: 144, 64: 272, 96: 400}
PLANAR_LM = (32, 64)   # key widths served by the planar compression GEMM


def planar_np(n):
    return -(-n // 128) * 128


def h_planes(H, stream=None):
    """(rows, 4 np) uint8 byte planes of H (the planar compression's A operand)."""
    rows, n = H.shape
    hp = torch.empty((rows, 4 * planar_np(n)), dtype=torch.uint8, device=H.device)
    _lib.call("zpir_h_planes", _lib.ptr(H), rows, n, _lib.ptr(hp), _s(stream))
    return hp


def build_bcp(cko, lm, stream=None, out=None):
    """cko (n, lm) or (nq, n, lm) int32 -> (nq, 4 lm, np) uint8 ck_o byte rows."""
    c = cko if cko.dim() == 3 else cko.unsqueeze(0)
    nq, n, _ = c.shape
    if out is None:
        out = torch.empty((nq, 4 * lm, planar_np(n)), dtype=torch.uint8, device=cko.device)
    _lib.call("zpir_build_bcp", _lib.ptr(c), n, lm, nq, _lib.ptr(out), _s(stream))
    return out


def umma_answer_rows_planar(hp, n, bp, lm, out=None, stream=None, ctas=0):
    """z (nq, rows, lm + 4) from H planes and ck_o byte rows."""
    rows = hp.shape[0]
    nq = bp.shape[0]
    if out is None:
        out = torch.empty((nq, rows, lm + 4), dtype=torch.int32, device=hp.device)
    _lib.call("zpir_umma_answer_rows_planar", _lib.ptr(hp), rows, n, _lib.ptr(bp), lm, nq, lm + 4,
              _lib.ptr(out), ctas, _s(stream))
    return out


def query_planes(qu_dev, prow, stream=None, planes=None):
    nvec, ld = qu_dev.shape
    if planes is None:
        planes = torch.empty((prow, ld), dtype=torch.uint8, device=qu_dev.device)
    _lib.call("zpir_query_planes", _lib.ptr(qu_dev), ld, nvec, _lib.ptr(planes), prow, _s(stream))
    return planes


def umma_gemv(dbt, planes, nvec, out=None, stream=None, ctas=0):
    rows, ld = dbt.shape
    if out is None:
        out = torch.empty((nvec, rows), dtype=torch.int32, device=dbt.device)
    _lib.call("zpir_umma_gemv", _lib.ptr(dbt), rows, ld, _lib.ptr(planes), nvec, _lib.ptr(out),
              ctas, _s(stream))
    return out


def umma_global_hint(dbt, A_dev, n, qmask, stream=None):
    rows, ld = dbt.shape
    ap = torch.empty((4 * n, ld), dtype=torch.uint8, device=dbt.device)
    _lib.call("zpir_build_aplanes", _lib.ptr(A_dev), ld, A_dev.shape[1], n, _lib.ptr(ap), _s(stream))
    H = torch.empty((rows, n), dtype=torch.int32, device=dbt.device)
    _lib.call("zpir_umma_global_hint", _lib.ptr(dbt), rows, ld, _lib.ptr(ap), n, _lib.ptr(H), qmask,
              _s(stream))
    return H


def build_bc(cko, lm, stream=None, bc=None):
    n = cko.shape[0]
    nb = UMMA_NB[lm]
    if bc is None:
        bc = torch.empty((nb, 4 * n), dtype=torch.uint8, device=cko.device)
    _lib.call("zpir_build_bc", _lib.ptr(cko), n, lm, nb, _lib.ptr(bc), _s(stream))
    return bc


def umma_answer_rows(H, bc, b, qmask, lm, out=None, stream=None, ctas=0):
    rows, n = H.shape
    if out is None:
        out = torch.empty((rows, lm + 4), dtype=torch.int32, device=H.device)
    _lib.call("zpir_umma_answer_rows", _lib.ptr(H), rows, n, _lib.ptr(bc), bc.shape[0],
              _lib.ptr(b) if b is not None else None,
              qmask, lm + 4, _lib.ptr(out), ctas, _s(stream))
    return out


def build_bc_batch(cko_all, lm, stream=None):
    """cko_all (nq, n, lm) int32 -> (nq, nb, 4n) uint8 stacked operands."""
    nq, n, _ = cko_all.shape
    nb = UMMA_NB[lm]
    bc = torch.empty((nq, nb, 4 * n), dtype=torch.uint8, device=cko_all.device)
    _lib.call("zpir_build_bc_batch", _lib.ptr(cko_all), n, lm, nb, nq, _lib.ptr(bc), _s(stream))
    return bc


def umma_answer_rows_batch(H, bc, lm, stream=None):
    rows, n = H.shape
    nq, nb, _ = bc.shape
    z = torch.empty((nq, rows, lm + 4), dtype=torch.int32, device=H.device)
    _lib.call("zpir_umma_answer_rows_batch", _lib.ptr(H), rows, n, _lib.ptr(bc), nb, nq, lm + 4,
              _lib.ptr(z), _s(stream))
    return z


_KEY_TABLES = {}
_KEY_TABLES_LOCK = threading.Lock()


def _key_tables(kctxs, nchunks, dev):
    """Per-query modulus tables of a batch (stacked moduli, R^k tables, -m^-1
    mod 2^32, R < 2m flags) on the device, cached per key sequence: building
    them from host lists would synchronise the stream on every batch."""
    key = (tuple(id(k) for k in kctxs), nchunks, str(dev))
    with _KEY_TABLES_LOCK:
        ent = _KEY_TABLES.get(key)
        if ent is None:
            if len(_KEY_TABLES) > 256:
                _KEY_TABLES.clear()
            mods = torch.stack([k.d_m for k in kctxs])
            rpows = torch.stack([k.d_rpow(nchunks) for k in kctxs])
            nps = torch.tensor(np.array([k.cm.np for k in kctxs], dtype=np.uint32).view(np.int32),
                               device=dev)
            f0 = torch.tensor([1 if k.cm.R < 2 * k.m else 0 for k in kctxs], dtype=torch.uint8,
                              device=dev)
            ent = _KEY_TABLES[key] = (mods, rpows, nps, f0, list(kctxs))
        return ent[:4]


def answer_groups_batch(z, b, qmask, d1, cap, groups, kctxs, t_ld, stream=None, stride=1):
    """z (nq, rows, lm+4), b (nq, rows); per-query Montgomery contexts."""
    nq, rows, wz = z.shape
    lm = kctxs[0].lm
    nchunks = max(2, -(-(stride * cap + lm + 4) // lm))
    dev = z.device
    mods, rpows, nps, f0 = _key_tables(kctxs, nchunks, dev)
    t = torch.empty((nq, groups, t_ld), dtype=torch.int32, device=dev)
    _lib.call("zpir_answer_groups_batch", _lib.ptr(z), rows * wz, _lib.ptr(b), b.shape[1], qmask, d1,
              cap, groups, lm, _lib.ptr(mods), _lib.ptr(nps), _lib.ptr(rpows), nchunks, _lib.ptr(f0),
              _lib.ptr(t), t_ld, nq, stride, _s(stream))
    return t


# ---- slot-decomposed hints / incremental update ------------------------------

def multiexp_rows(bases, E, row_ids, rows, rs, bs, ls, elimbs, kctx, out, keep_mont, stream=None):
    n = bases.shape[0]
    l2 = kctx.l2
    ws_bytes = int(_lib.lib().zpir_multiexp_workspace_bytes(n, rows, elimbs, l2))
    ws = torch.empty(ws_bytes // 4 + 64, dtype=torch.int32, device=bases.device)
    _lib.call("zpir_multiexp_rows", _lib.ptr(bases), n, _lib.ptr(E),
              _lib.ptr(row_ids) if row_ids is not None else None, rows, rs, bs, ls, elimbs, l2,
              _lib.ptr(kctx.d_m2), kctx.c2.np, _lib.ptr(kctx.d_r2sq), _lib.ptr(kctx.d_one2),
              1 if keep_mont else 0, _lib.ptr(out), _lib.ptr(ws), ws_bytes, _s(stream))
    return out


def slot_combine(W, cap, group_ids, ngroups, kctx, out, gamma=1 << 32, stream=None):
    gw = np.frombuffer(int(gamma).to_bytes(32, "little"), dtype="<u4").copy()
    _lib.call("zpir_slot_combine", _lib.ptr(W), cap,
              _lib.ptr(group_ids) if group_ids is not None else None, ngroups, kctx.l2,
              _lib.ptr(kctx.d_m2), kctx.c2.np, gw.ctypes.data_as(ctypes.c_void_p),
              int(gamma).bit_length(), _lib.ptr(out), _s(stream))
    return out


def slot_combine_many(jobs, cap, group_ids, ngroups, gamma=1 << 32, stream=None):
    """slot_combine for several clients of one key width in one launch.
    jobs: [(W, kctx, out)]."""
    import ctypes
    c = len(jobs)
    arr = lambda vals: (ctypes.c_uint64 * c)(*vals)  # noqa: E731
    W = arr([w.data_ptr() for w, _, _ in jobs])
    N = arr([k.d_m2.data_ptr() for _, k, _ in jobs])
    out = arr([o.data_ptr() for _, _, o in jobs])
    np_ = (ctypes.c_uint32 * c)(*[k.c2.np for _, k, _ in jobs])
    gw = np.frombuffer(int(gamma).to_bytes(32, "little"), dtype="<u4").copy()
    _lib.call("zpir_slot_combine_many", c, W, N, np_, out, cap,
              _lib.ptr(group_ids) if group_ids is not None else None, ngroups, jobs[0][1].l2,
              gw.ctypes.data_as(ctypes.c_void_p), int(gamma).bit_length(), _s(stream))
    return [o for _, _, o in jobs]


def answer_general(z, b, qmask, d1, cap, groups, kctx, gamma, t_ld, stream=None):
    """Group stage for a general batch scale gamma (per-row weights)."""
    lm = kctx.lm
    ctab = kctx.d_gamma_table(gamma, cap)
    w = torch.empty((d1, lm), dtype=torch.int32, device=z.device)
    t = torch.empty((groups, t_ld), dtype=torch.int32, device=z.device)
    _lib.call("zpir_answer_general", _lib.ptr(z), _lib.ptr(b), qmask, d1, cap, groups, lm,
              _lib.ptr(kctx.d_m), kctx.cm.np, _lib.ptr(ctab), _lib.ptr(w), _lib.ptr(t), t_ld,
              _s(stream))
    return t


def answer_groups_strided(z, b, qmask, d1, cap, groups, kctx, t_ld, stride, stream=None):
    """Positional group stage (gamma = 2^(32 stride)) for one query."""
    lm = kctx.lm
    nchunks = max(2, -(-(stride * cap + lm + 4) // lm))
    rpow = kctx.d_rpow(nchunks)
    nps = torch.tensor(np.array([kctx.cm.np], dtype=np.uint32).view(np.int32), device=z.device)
    f0 = torch.tensor([1 if kctx.cm.R < 2 * kctx.m else 0], dtype=torch.uint8, device=z.device)
    t = torch.empty((groups, t_ld), dtype=torch.int32, device=z.device)
    rows, wz = z.shape
    _lib.call("zpir_answer_groups_batch", _lib.ptr(z), rows * wz, _lib.ptr(b), b.shape[-1], qmask,
              d1, cap, groups, lm, _lib.ptr(kctx.d_m), _lib.ptr(nps), _lib.ptr(rpow), nchunks,
              _lib.ptr(f0), _lib.ptr(t), t_ld, 1, stride, _s(stream))
    return t


def rows_differ(a, b, stream=None):
    rows, ld = a.shape
    flags = torch.empty(rows, dtype=torch.int32, device=a.device)
    _lib.call("zpir_rows_differ", _lib.ptr(a), _lib.ptr(b), rows, ld, _lib.ptr(flags), _s(stream))
    return flags


def move_rows(src, dst, ids, scatter, stream=None):
    """Row gather (dst[i] = src[ids[i]]) or scatter (dst[ids[i]] = src[i])."""
    pitch = src.shape[1] * src.element_size()
    _lib.call("zpir_move_rows", _lib.ptr(src), _lib.ptr(dst), pitch, _lib.ptr(ids), ids.numel(),
              1 if scatter else 0, _s(stream))
    return dst


def pow8_table(bases, kctx, stream=None):
    n = bases.shape[0]
    P = torch.empty((4 * n, kctx.l2), dtype=torch.int32, device=bases.device)
    _lib.call("zpir_pow8_table", _lib.ptr(bases), n, kctx.l2, _lib.ptr(kctx.d_m2), kctx.c2.np,
              _lib.ptr(kctx.d_r2sq), _lib.ptr(P), _s(stream))
    return P


def slot_fixed(P, n, E, rs, row_ids, rows, kctx, W, stream=None):
    _lib.call("zpir_slot_fixed", _lib.ptr(P), n, _lib.ptr(E), rs,
              _lib.ptr(row_ids) if row_ids is not None else None, rows, kctx.l2,
              _lib.ptr(kctx.d_m2), kctx.c2.np, _lib.ptr(kctx.d_one2), _lib.ptr(W), _s(stream))
    return W


def slot_fixed_tc(P, n, E, rs, rows, kctx, W, stream=None):
    """slot_fixed (all rows) with the bucket updates on the tensor cores."""
    _lib.call("zpir_slot_fixed_tc", _lib.ptr(P), n, _lib.ptr(E), rs, rows, kctx.l2,
              _lib.ptr(kctx.d_m2), kctx.c2.np, _lib.ptr(kctx.d_one2), _lib.ptr(W), _s(stream))
    return W


def slot_fixed_tc_many(jobs, n, E, rs, rows, rid=None, stream=None):
    """slot_fixed_tc for several clients in one launch (blockIdx.y = client).

    jobs: [(P, kctx, W)] -- client table P (4n x 128 limbs), its key context and
    its output rows W (Montgomery form); rows r < rows read exponent row
    rid[r] (or r) of E and write W[rid[r]] (or W[r])."""
    import ctypes
    c = len(jobs)
    arr = lambda vals: (ctypes.c_uint64 * c)(*vals)  # noqa: E731
    P = arr([p.data_ptr() for p, _, _ in jobs])
    N = arr([k.d_m2.data_ptr() for _, k, _ in jobs])
    one = arr([k.d_one2.data_ptr() for _, k, _ in jobs])
    W = arr([w.data_ptr() for _, _, w in jobs])
    np_ = (ctypes.c_uint32 * c)(*[k.c2.np for _, k, _ in jobs])
    _lib.call("zpir_slot_fixed_tc_many", c, P, N, np_, one, W, n, _lib.ptr(E), rs,
              _lib.ptr(rid) if rid is not None else None, rows, _s(stream))
    return [w for _, _, w in jobs]


def slot_fixed_tc_workspace(n, rows, clients):
    return _lib.lib().zpir_slot_fixed_tc_workspace(n, rows, clients)


def groups_z(z, d1, cap, groups, lm, d_m, d_np, d_rpow, nchunks, d_f0, tz, t_ld, stream=None,
             stride=1):
    rows, wz = z.shape[-2], z.shape[-1]
    nq = 1 if z.dim() == 2 else z.shape[0]
    _lib.call("zpir_groups_z", _lib.ptr(z), rows * wz, d1, cap, groups, lm, _lib.ptr(d_m),
              _lib.ptr(d_np), _lib.ptr(d_rpow), nchunks, _lib.ptr(d_f0), _lib.ptr(tz), t_ld, nq,
              stride, _s(stream))
    return tz


def groups_finish(tz, b, qmask, d1, cap, groups, lm, d_m, t, t_ld, stream=None, stride=1):
    nq = 1 if b.dim() == 1 or b.shape[0] == 1 else b.shape[0]
    _lib.call("zpir_groups_finish", _lib.ptr(tz), _lib.ptr(b), b.shape[-1], qmask, d1, cap, groups,
              lm, _lib.ptr(d_m), _lib.ptr(t), t_ld, nq, stride, _s(stream))
    return t


# ---- device ChaCha20 (prg.py) -------------------------------------------------

def chacha_words32(seed: bytes, domain: int, index: int, rows, cols, out, ld, mask, stream=None):
    import hashlib
    key = hashlib.sha256(seed).digest()
    iv = bytes([domain]) + int(index).to_bytes(15, "little")
    _lib.call("zpir_chacha_words32", key, iv, rows, cols, _lib.ptr(out), ld, mask, _s(stream))
    return out


def chacha_below(seed: bytes, domain: int, query_index: int, n: int, d_bound, bound: int, limbs,
                 stream=None):
    """(n, limbs) int32: Stream(seed, domain, (qi << 32) | k).below(bound)."""
    import hashlib
    key = hashlib.sha256(seed).digest()
    bits = (bound - 1).bit_length()
    out = torch.empty((n, limbs), dtype=torch.int32, device=d_bound.device)
    _lib.call("zpir_chacha_below", key, domain, query_index, n, _lib.ptr(d_bound), limbs, bits,
              _lib.ptr(out), _s(stream))
    return out


def digits_to_limbs(digits, nl, out, stream=None):
    count, ndig = digits.shape
    _lib.call("zpir_digits_to_limbs", _lib.ptr(digits), count, ndig, _lib.ptr(out), nl, _s(stream))
    return out


def limbs_to_digits(limbs, nl, digits, stream=None):
    count, ld = limbs.shape
    _lib.call("zpir_limbs_to_digits", _lib.ptr(limbs), count, nl, ld, _lib.ptr(digits),
              digits.shape[1], _s(stream))
    return digits


def event_record(event, stream):
    """Timing event record that also fires inside replayed CUDA graphs."""
    _lib.call("zpir_event_record", ctypes.c_void_p(event.cuda_event), _s(stream))


def stream_wait_event(stream, event):
    """Stream waits for an event; an external wait node when captured."""
    _lib.call("zpir_stream_wait_event", _s(stream), ctypes.c_void_p(event.cuda_event))


def graph_launch(graph_exec: int, stream):
    _lib.call("zpir_graph_launch", ctypes.c_void_p(graph_exec), _s(stream))


def h2d_async(dst, src_pinned, stream):
    """Raw cudaMemcpyAsync pinned host -> device (same byte size)."""
    _lib.call("zpir_memcpy_async", _lib.ptr(dst), _lib.ptr(src_pinned),
              src_pinned.numel() * src_pinned.element_size(), 0, _s(stream))


def d2h_async(dst_pinned, src, stream):
    _lib.call("zpir_memcpy_async", _lib.ptr(dst_pinned), _lib.ptr(src),
              src.numel() * src.element_size(), 1, _s(stream))


# -- bulk host -> device upload of a database ----------------------------------------

_UPLOAD_CHUNK = 64 << 20
_UPLOAD_MIN = 16 << 20
_UPLOAD_LOCK = threading.Lock()
_UPLOAD_STAGES = {}
_UPLOAD_POOL = None


UPLOAD_THREADS = None     # host threads for staging copies (None: min(8, cpu count))


def _upload_threads() -> int:
    import os
    return UPLOAD_THREADS if UPLOAD_THREADS is not None else max(1, min(8, os.cpu_count() or 1))


def host_threads() -> int:
    """Threads for host-side staging copies (UPLOAD_THREADS, else <= 8)."""
    return _upload_threads()


def upload_bytes(a: np.ndarray, dev, stream) -> torch.Tensor:
    """A host byte array (a database, ~1 GiB) -> a device uint8 tensor of the
    same shape, queued on `stream`. Pageable copies go through the driver's
    single-threaded bounce buffer (~12 GB/s on the B200 hosts); here the host
    side copies chunks into two pinned 64 MB stages split over threads (numpy
    copies release the GIL) while the previous stage's DMA runs."""
    a = np.ascontiguousarray(a, dtype=np.uint8)
    out = torch.empty(a.shape, dtype=torch.uint8, device=dev)
    nthreads = _upload_threads()
    if a.nbytes < _UPLOAD_MIN or nthreads == 0:
        import warnings
        with warnings.catch_warnings():  # read-only numpy views are only read here
            warnings.simplefilter("ignore", UserWarning)
            with torch.cuda.stream(stream):
                out.copy_(torch.from_numpy(a))
        return out
    global _UPLOAD_POOL
    flat = a.reshape(-1)
    o = out.view(-1)
    with _UPLOAD_LOCK:
        if _UPLOAD_POOL is None or _UPLOAD_POOL[0] != nthreads:
            from concurrent.futures import ThreadPoolExecutor
            if _UPLOAD_POOL is not None:
                _UPLOAD_POOL[1].shutdown(wait=False)
            _UPLOAD_POOL = (nthreads, ThreadPoolExecutor(nthreads, thread_name_prefix="zpir-upload"))
        pool = _UPLOAD_POOL[1]
        key = str(dev)
        if key not in _UPLOAD_STAGES:
            _UPLOAD_STAGES[key] = [
                (torch.empty(_UPLOAD_CHUNK, dtype=torch.uint8).pin_memory(),
                 torch.cuda.Event()) for _ in range(2)]
        stages = _UPLOAD_STAGES[key]
        for i, off in enumerate(range(0, flat.size, _UPLOAD_CHUNK)):
            buf, ev = stages[i % 2]
            ev.synchronize()                  # this stage's previous DMA is done
            n = min(_UPLOAD_CHUNK, flat.size - off)
            st = buf.numpy()
            cuts = [n * t // nthreads for t in range(nthreads + 1)]
            list(pool.map(
                lambda t: np.copyto(st[cuts[t]:cuts[t + 1]], flat[off + cuts[t]:off + cuts[t + 1]]),
                range(nthreads)))
            with torch.cuda.stream(stream):
                o[off:off + n].copy_(buf[:n], non_blocking=True)
            ev.record(stream)
        # the stages may be reused by the next upload only after these copies
        for buf, ev in stages:
            ev.synchronize()
    return out
