#!/usr/bin/env python
"""ZipPIR online-answer throughput on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl b200|reference]
    python -m torch.distributed.run --nnodes=1 --nproc-per-node N \
        --master-addr 127.0.0.1 --master-port P bench.py --gpus N ...

Workload (BASELINE.json configs[1]): 1 GiB DB per GPU, d0 = 32768 records x
32768 output rows (u8, uniform, seeded), LWE n = 1024, q = 2^32, 2048-bit
Paillier modulus; one query per step: b = DB qu mod 2^32, the compression
t_g = (sum_j 2^(32j)(b + H ck_o)) mod m for all d1' = 521 groups. With N
GPUs the DB is N GiB, row-sharded (group aligned, 1 GiB per GPU: weak
scaling) and the per-shard t is gathered over NCCL.

value   = DB bytes (all ranks) / device time per answer, inputs resident in
          HBM; the DB (1 GiB) exceeds L2 (126 MB), so no flush is needed.
e2e     = same metric through protocol.respond() with host inputs
          (numpy qu0, Python-int ck_o) and a host ResponseMessage.
roofline: the GEMV kernel, algorithmic bytes d0*d1 + 4 d0 + 4 d1 per launch
          over its CUDA-event time, against MEASURED_PEAKS.json hbm_gbs.
cpu_baseline: the reference's own algorithm (oracle/ref_port.py: float64
          BLAS GEMV + 240-prime RNS) on a bounded row sample, rank 0, N=1.
"""

import argparse
import json
import os
import random
import statistics
import subprocess
import sys
import tempfile
import threading
import time

import numpy as np

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

D0 = 32768
D1 = 32768
N_LWE = 1024
BITS = 2048
CAP = 63
CPU_SAMPLE_ROWS = 32 * CAP  # 2016 DB rows = 32 groups


def _args():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=200)
    ap.add_argument("--warmup", type=int, default=20)
    ap.add_argument("--impl", default="b200", choices=["b200", "reference"])
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--ref-rows", type=int, default=0,
                    help="reference arm: serve only this many DB rows (0 = the whole config)")
    ap.add_argument("--dist-backend", default="nccl",
                    help="process-group backend for N > 1 (gloo only to exercise the multi-rank "
                         "code path with several ranks on one GPU; never for numbers)")
    ap.add_argument("--no-single-thread", action="store_true",
                    help="reference arm: skip the single-thread figure")
    ap.add_argument("--e2e-steps", type=int, default=50)
    ap.add_argument("--no-extra-e2e", action="store_true",
                    help="skip the wire / C-ABI e2e variants")
    ap.add_argument("--workload", default="1g", choices=["1g", "batch64", "8g", "hint", "update", "tiny"],
                    help="1g: BASELINE configs[1] (default, the driver's line); batch64: "
                         "configs[3]; 8g: configs[2] (92682^2, strong-scaled over --gpus); "
                         "hint: configs[4] offline hint generation")
    return ap.parse_args()


def _dist_env():
    rank = int(os.environ.get("RANK", "0"))
    world = int(os.environ.get("WORLD_SIZE", "1"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    return rank, world, local


# -- seeded inputs (no oracle on the product path) ---------------------------

def _is_prime(x):
    for p in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37):
        if x % p == 0:
            return x == p
    d, s = x - 1, 0
    while d % 2 == 0:
        d //= 2
        s += 1
    for a in (2, 3, 5, 7, 11, 13, 17, 19, 23, 29, 31, 37, 41):
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


def paillier_modulus(bits, seed):
    """m = p q with two seeded bits/2-bit primes (same recipe as paillier.py:69-86)."""
    import math
    rng = random.Random(seed)
    half = bits // 2
    while True:
        ps = []
        for _ in range(2):
            x = rng.randrange(1 << (half - 1), 1 << half) | 1
            while not _is_prime(x):
                x += 2
            ps.append(x)
        p, q = ps
        m = p * q
        if p != q and m.bit_length() == bits and math.gcd(m, (p - 1) * (q - 1)) == 1:
            return m


def db_slice(rank, rows):
    return np.frombuffer(np.random.default_rng(7 + rank).bytes(D0 * rows),
                         dtype=np.uint8).reshape(D0, rows)


# -- clocks --------------------------------------------------------------------

class ClockSampler:
    FIELDS = ("index,clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.active,"
              "clocks_event_reasons.hw_slowdown,clocks_event_reasons.hw_thermal_slowdown,"
              "clocks_event_reasons.sw_thermal_slowdown,clocks_event_reasons.sw_power_cap")

    def __init__(self, index):
        self.index = index
        self.proc = None
        self.path = None

    def start(self):
        try:
            fd, self.path = tempfile.mkstemp(suffix=".csv")
            os.close(fd)
            self.proc = subprocess.Popen(
                ["nvidia-smi", "-i", str(self.index), f"--query-gpu={self.FIELDS}",
                 "--format=csv,noheader,nounits", "-lms", "100"],
                stdout=open(self.path, "w"), stderr=subprocess.DEVNULL)
        except Exception:
            self.proc = None

    def stop(self):
        if self.proc is None:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["nvidia-smi unavailable"]}
        self.proc.terminate()
        self.proc.wait(timeout=5)
        sm, smax, reasons = [], [], set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        for line in open(self.path):
            f = [x.strip() for x in line.split(",")]
            if len(f) < 9:
                continue
            try:
                sm.append(float(f[1]))
                smax.append(float(f[2]))
            except ValueError:
                continue
            for nm, v in zip(names, f[5:9]):
                if v.lower().startswith("active"):
                    reasons.add(nm)
        os.unlink(self.path)
        return {"sm_mhz": statistics.median(sm) if sm else None,
                "sm_max_mhz": max(smax) if smax else None,
                "samples": len(sm), "reasons": sorted(reasons)}


def _peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md)"


def _traffic():
    p = os.path.join(ROOT, "profiles", "gemv_traffic.json")
    try:
        return json.load(open(p)).get("bytes_per_launch")
    except Exception:
        return None


def _config(world):
    """The workload description, identical in both arms (driver same_config)."""
    return {"workload": "BASELINE configs[1]: 1 GiB DB per GPU (32768 x 32768 u8), "
                        "n=1024, q=2^32, 2048-bit Paillier, single query, SEPARATE",
            "d0": D0, "d1": D1 * world, "groups": -(-(D1 * world) // CAP), "n": N_LWE,
            "paillier_bits": BITS, "queries_per_step": 1,
            "l2": "no flush: the DB (1 GiB per GPU) exceeds L2 (126 MB) and the host LLC"}


def _threads(n):
    try:
        from threadpoolctl import threadpool_limits
        threadpool_limits(n)
    except Exception:
        pass


def _cpu_query(m):
    rng = np.random.default_rng(11)
    qu = rng.integers(0, 1 << 32, D0, dtype=np.uint64)
    r = random.Random(12)
    return qu, [r.randrange(m) for _ in range(N_LWE)]


def _port_state(rows, d0=D0, seed_rank=0):
    """The reference's ServerGlobalState built its own way (oracle/ref_port.py:
    float64 GEMMs for H, H_scaled, 240-prime residues, the centered float64
    DB copy) over DB rows [0, rows); A from oracle/ref's ChaCha20."""
    from oracle import ref, ref_port
    db = db_slice(seed_rank, D1)[:, :rows] if d0 == D0 else None
    db = np.ascontiguousarray(db)
    A = ref.public_matrix(b"\x00" * 16, d0, N_LWE, 1 << 32)
    return ref_port.PortState(db, A, CAP)


def cpu_baseline(m, repeats=7):
    """Bounded sample beside the B200 line: the reference algorithm on
    CPU_SAMPLE_ROWS of the 32768 DB rows, all host cores."""
    _threads(os.cpu_count())
    rows = CPU_SAMPLE_ROWS
    st = _port_state(rows)
    qu, ck_o = _cpu_query(m)
    times = []
    for _ in range(repeats):
        t0 = time.perf_counter()
        st.respond_t(qu, ck_o, m)
        times.append(time.perf_counter() - t0)
    best = min(times)
    return {"value": D0 * rows / best / 1e9, "unit": "GB/s", "cores": os.cpu_count(),
            "kind": "port",
            "sample": f"{rows} of {D1} DB rows ({rows // CAP} groups) x d0={D0}, n={N_LWE}, "
                      f"{BITS}-bit m; reference algorithm (centered float64 BLAS GEMV + "
                      f"240x27-bit RNS matvec + Garner), best of {repeats}, "
                      f"median {statistics.median(times) * 1e3:.1f} ms",
            "best_s": best}


def run_reference(args):
    """The reference arm: the reference's own CPU algorithm for respond()
    (oracle/ref_port.py, bit-exact with the reference's goldens) on the
    B200 arm's config, all host cores; exactly --warmup untimed and --steps
    timed respond()s. At N = 1 the whole configs[1] DB (32768 x 32768) is
    served; at N > 1 (N GiB) a 1 GiB row slice is timed and the metric is
    per DB byte of that slice. Then the same respond() single-threaded
    (OPENBLAS_NUM_THREADS = 1, the paper's methodology)."""
    rank, world, _ = _dist_env()
    if rank != 0:
        return
    _threads(os.cpu_count())
    m = paillier_modulus(BITS, 2048)
    rows = args.ref_rows or D1
    t0 = time.perf_counter()
    st = _port_state(rows)
    setup_s = time.perf_counter() - t0
    qu, ck_o = _cpu_query(m)
    for _ in range(args.warmup):
        st.respond_t(qu, ck_o, m)
    times = []
    for _ in range(args.steps):
        t1 = time.perf_counter()
        st.respond_t(qu, ck_o, m)
        times.append(time.perf_counter() - t1)
    dt = statistics.mean(times)
    v = D0 * rows / dt / 1e9
    one = None
    if not args.no_single_thread:
        _threads(1)
        t1s = []
        for _ in range(2):
            t1 = time.perf_counter()
            st.respond_t(qu, ck_o, m)
            t1s.append(time.perf_counter() - t1)
        _threads(os.cpu_count())
        one = {"value": D0 * rows / min(t1s) / 1e9, "unit": "GB/s", "cores": 1,
               "ms_per_step": min(t1s) * 1e3, "note": "OPENBLAS_NUM_THREADS=1, best of 2"}
    whole = rows == D1 * world
    sample = (f"{'all' if whole else rows} of {D1 * world} DB rows x d0={D0} per step, "
              f"n={N_LWE}, {BITS}-bit m: the reference's respond() algorithm (oracle/ref_port.py: "
              "centered float64 BLAS GEMV + 240x27-bit-prime RNS matvec + Garner + scaled_b), "
              f"{os.cpu_count()} host threads")
    print(json.dumps({
        "impl": "reference", "metric": "online server throughput (DB GB/s per query)",
        "value": v, "unit": "GB/s", "n_gpus": world, "steps": args.steps, "warmup": args.warmup,
        "ms_per_step": dt * 1e3, "higher_is_better": True, "scaling": "weak",
        "vs_baseline": None, "dtype": "u8xu32 mod 2^32 / 2048-bit (float64-exact + RNS on CPU)",
        "data": "synthetic (seeded uniform u8 DB, uniform qu0 / ck_o, seeded Paillier modulus)",
        "config": _config(world),
        "cpu_baseline": {"value": v, "unit": "GB/s", "cores": os.cpu_count(), "kind": "port",
                         "sample": sample},
        "e2e": {"value": v, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
        "single_thread": one, "setup_s": setup_s,
        "ms_per_step_median": statistics.median(times) * 1e3,
        "cpu_model": _cpu_model(),
    }), flush=True)


def cpu_hint_baseline(db, m, nentries=None):
    """Reference-equivalent hint cost on the host: the reference's windowed
    multiexp (paillier.py:134-193) restated over libgmp (oracle/c, the
    library gmpy2 wraps) on `nentries` real 1 GiB hint entries (exponents from
    the oracle's H of the first groups, ck_r from the oracle's ChaCha20),
    one entry per host thread in parallel; extrapolated x d1' per client and
    x 256 clients as the reference's bench.py:183-190 does."""
    from oracle import c as oc, ref
    threads = os.cpu_count()
    nentries = nentries or threads
    A = ref.public_matrix(b"\x00" * 16, D0, N_LWE, 1 << 32)
    H = oc.hint_rows(db, A, 0, nentries * CAP)
    E = oc.scaled_exponents(H, CAP)
    m2 = m * m
    ck_r = ref.derive_ck_r(m2, b"\x05" * 16, 0, N_LWE)
    t0 = time.perf_counter()
    oc.multiexp_rows(ck_r, E, m2)
    wall = time.perf_counter() - t0
    per_entry_core = wall * min(threads, nentries) / nentries     # one core, one entry
    groups = -(-D1 // CAP)
    per_client = per_entry_core * groups / threads
    return {"value": per_client, "unit": "s per client (all host cores)", "cores": threads,
            "kind": "port",
            "sample": f"{nentries} hint entries (groups 0..{nentries - 1}, 1024 exponents of "
                      f"2016 bits, 4096-bit m^2) by the reference's w=6 windowed multiexp over "
                      f"libgmp, {threads} threads; {per_entry_core:.2f} s per entry per core, "
                      f"x {groups} entries per client / {threads} cores",
            "per_entry_core_s": per_entry_core, "clients_256_s": 256 * per_client}


def cpu_rebuild_baseline(db, rows=CPU_SAMPLE_ROWS):
    """The reference's full state rebuild (ServerGlobalState.__init__:
    float64 H GEMMs, H_scaled, residues, centered DB copy) on a row sample,
    extrapolated linearly to all 32768 rows."""
    _threads(os.cpu_count())
    from oracle import ref, ref_port
    A = ref.public_matrix(b"\x00" * 16, D0, N_LWE, 1 << 32)
    part = np.ascontiguousarray(db[:, :rows])
    t0 = time.perf_counter()
    ref_port.PortState(part, A, CAP)
    dt = time.perf_counter() - t0
    return dt * D1 / rows, f"{rows} of {D1} DB rows, x{D1 / rows:.2f}"


def _cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except OSError:
        pass
    return None


# -- B200 path -----------------------------------------------------------------

def run_b200(args):
    import torch
    rank, world, local = _dist_env()
    local %= max(1, torch.cuda.device_count())     # (gloo code-path runs: ranks share a GPU)
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    group = None
    if world > 1:
        import torch.distributed as dist
        if args.dist_backend == "nccl":
            dist.init_process_group("nccl", device_id=dev)
        else:
            dist.init_process_group(args.dist_backend)
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import _lib, build as zb
    from paper_2603_09190_b200.bigint import ints_to_limbs, key_ctx
    from paper_2603_09190_b200.shard import ShardedServer, shard_bounds
    zb.build()
    _lib.load()

    d1_total = D1 * world
    params = z.ProtocolParams(z.LweParams(N_LWE, 1 << 32, 256, 6.4), D0, d1_total, BITS)
    bounds = shard_bounds(d1_total, params.capacity, world)
    lo, hi, g_lo, g_hi = bounds[rank]
    t0 = time.perf_counter()
    db = db_slice(rank, hi - lo)
    srv = ShardedServer(params, db, rank, world, group)
    st = srv.state
    setup_s = time.perf_counter() - t0
    m = paillier_modulus(BITS, 2048)
    kctx = key_ctx(m, dev)
    pk = z.PaillierPublicKey(m, m.bit_length())
    reg = z.ClientRegistration(pk, b"\x05" * 16, z.client_id_of(pk))
    stream = torch.cuda.current_stream(dev)

    # per-client hint (offline): one device multi-exponentiation, all groups;
    # the first call also loads the kernels and grows the memory pool
    reg.hints[0] = z.hint(st, reg, 0)
    torch.cuda.synchronize()
    th = time.perf_counter()
    reg.hints[0] = z.hint(st, reg, 0)
    torch.cuda.synchronize()
    hint_s = time.perf_counter() - th

    rng = np.random.default_rng(100 + rank)
    qu = rng.integers(0, 1 << 32, D0, dtype=np.uint64)
    r = random.Random(200)
    ck_o = [r.randrange(m) for _ in range(N_LWE)]
    lay = st.layout
    q32 = np.zeros(lay.ld, dtype=np.uint32)
    q32[:D0] = qu.astype(np.uint32)
    plan = st.answer_plan(kctx, kctx.lm)
    plan.qu.copy_(torch.from_numpy(q32.view(np.int32)).to(dev).reshape(1, lay.ld))
    plan.cko.copy_(torch.from_numpy(ints_to_limbs(ck_o, kctx.lm).view(np.int32)).to(dev))

    def step():
        plan.run("full", stream)
        if world > 1:
            from paper_2603_09190_b200.shard import gather_groups
            with torch.cuda.stream(stream):
                gather_groups(plan.t, bounds, rank)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731

    def timed(fn, steps):
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        e0.record(stream)
        for _ in range(steps):
            fn()
        e1.record(stream)
        torch.cuda.synchronize()
        return e0.elapsed_time(e1) / steps

    for _ in range(max(args.warmup, 3)):
        step()
        plan.run("gemv", stream)
        plan.run("compress", stream)
    if world > 1:
        import torch.distributed as dist
    clocks = ClockSampler(local)
    clocks.start()
    # burn-in so the sampled clocks reflect steady load (not part of timing)
    tb = time.perf_counter()
    while time.perf_counter() - tb < 1.5:
        for _ in range(50):
            step()
        torch.cuda.synchronize()
    ms = timed(step, args.steps)
    # the GEMV (query planes + tcgen05 GEMV on SMs - COMPRESS_CTAS) inside the
    # full step, concurrent with the compression: events captured around it
    # in the step's graph, read after every replay
    # (steady state: each reading is the last of 20 back-to-back step replays)
    ge0, ge1 = plan.gemv_events
    se0, se1 = plan.side_events
    in_step, side_step = [], []
    plan.run("full_timed", stream)
    for i in range(12):
        for _ in range(20):
            plan.run("full_timed", stream)
        stream.synchronize()
        if i >= 2:
            in_step.append(ge0.elapsed_time(ge1))
            if plan.ctas > 0:
                side_step.append(se0.elapsed_time(se1))
    gemv_step_ms = statistics.mean(in_step)
    side_step_ms = statistics.mean(side_step) if side_step else None
    # the GEMV kernel alone (all SMs); and the compression half
    gemv_ms = timed(lambda: plan.run("gemv", stream), args.steps)
    comp_ms = timed(lambda: plan.run("compress", stream), args.steps)
    clk = clocks.stop()
    if world > 1:
        t = torch.tensor([ms, gemv_ms, comp_ms, gemv_step_ms], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms, gemv_ms, comp_ms, gemv_step_ms = t.tolist()

    # e2e through the public API (host buffers, H2D/D2H inside). N > 1: the
    # sharded server -- rank 0 receives the query, broadcasts qu0 + ck_o, every
    # rank answers its shard, the t rows are gathered to rank 0 (shard.py)
    qmsg = z.QueryMessage(reg.client_id, 0, z.SEPARATE, ck_o, qu)
    api = "paper_2603_09190_b200.respond()"
    if world == 1:
        for _ in range(3):
            z.respond(st, reg, qmsg)
        e2e_times = []
        for _ in range(args.e2e_steps):
            t1 = time.perf_counter()
            z.respond(st, reg, qmsg)
            e2e_times.append(time.perf_counter() - t1)
        e2e_s = statistics.mean(e2e_times)
    else:
        from paper_2603_09190_b200.shard import DeviceShard, ShardedPirServer
        from paper_2603_09190_b200.shard import shard_params
        api = "ShardedPirServer.respond() on rank 0 (broadcast, per-shard answer, NCCL gather)"
        local = DeviceShard(shard_params(params, hi - lo), None, state=st)
        sps = ShardedPirServer(params, None, local=local, hint_batch=1)
        if rank == 0:
            cid = sps.register(pk, reg.seed)
            sps.wait_for_hints(timeout=600)
            for _ in range(3):
                sps.respond(cid, qmsg)
            e2e_times = []
            for _ in range(args.e2e_steps):
                t1 = time.perf_counter()
                sps.respond(cid, qmsg)
                e2e_times.append(time.perf_counter() - t1)
            e2e_s = statistics.mean(e2e_times)
            sps.close()
        else:
            sps.join()
            sps.close()
            e2e_s = 0.0
        t = torch.tensor([e2e_s], dtype=torch.float64, device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        e2e_s = t.item()

    # the same answer through the wire front end (PirServer.handle_frame: query
    # frame bytes in, response frame bytes out) and through the host-buffer
    # C ABI handle (zpir_db_answer), single GPU only
    extra_e2e = {}
    if world == 1 and not args.no_extra_e2e:
        from paper_2603_09190_b200 import wire
        from paper_2603_09190_b200.dbapi import DeviceDatabase
        from paper_2603_09190_b200.server import PirServer
        srv_w = PirServer(params, None, state=st, hint_workers=1)
        srv_w.close()                      # no background hint jobs during timing
        srv_w.registrations[reg.client_id] = reg
        wl = wire.WireLayout(params)
        frame = wire.pack_frame(wire.MSG_QUERY, params.params_hash(),
                                wire.encode_query(wl, reg.client_id, 0, 0, ck_o, qu))[4:]
        for _ in range(3):
            rep = srv_w.handle_frame(frame)
        assert rep[5] == wire.MSG_RESPONSE_SEPARATE, rep[:64]
        tw = []
        for _ in range(args.e2e_steps):
            t1 = time.perf_counter()
            srv_w.handle_frame(frame)
            tw.append(time.perf_counter() - t1)
        wire_s = statistics.mean(tw)
        extra_e2e["e2e_wire"] = {"value": D0 * d1_total / wire_s / 1e9, "unit": "GB/s",
                                 "ms_per_step": wire_s * 1e3,
                                 "request_bytes": len(frame), "reply_bytes": len(rep),
                                 "api": "PirServer.handle_frame (query frame bytes -> response "
                                        "frame bytes, SEPARATE)"}
        del srv_w
        dd = DeviceDatabase(params, db)
        for _ in range(3):
            t_h = dd.answer(qu, ck_o, m)
        assert t_h == z.respond(st, reg, qmsg).t
        th_ = []
        for _ in range(args.e2e_steps):
            t1 = time.perf_counter()
            dd.answer(qu, ck_o, m)
            th_.append(time.perf_counter() - t1)
        # the bare C call a C / cgo / JNI caller makes: limb arrays already in
        # (pageable) host memory, t's limbs written back to host memory
        from paper_2603_09190_b200 import _lib
        from paper_2603_09190_b200.dbapi import _vp
        q_l, c_l, m_l, L_l = dd._query(qu, ck_o, m)
        t_l = np.empty((dd.groups, L_l), dtype=np.uint32)
        tc_ = []
        for i in range(3 + args.e2e_steps):
            t1 = time.perf_counter()
            _lib.call("zpir_db_answer", dd._h, _vp(q_l), _vp(c_l), _vp(m_l), L_l, _vp(t_l))
            if i >= 3:
                tc_.append(time.perf_counter() - t1)
        from paper_2603_09190_b200.bigint import limbs_to_ints
        assert limbs_to_ints(t_l) == t_h
        dd.close()
        h_s = statistics.mean(th_)
        c_s = statistics.mean(tc_)
        extra_e2e["e2e_c_abi"] = {"value": D0 * d1_total / h_s / 1e9, "unit": "GB/s",
                                  "ms_per_step": h_s * 1e3,
                                  "api": "zpir_db_answer (include/zippir_db.h): pageable host "
                                         "buffers, Python ints converted by dbapi.py",
                                  "call_only": {"value": D0 * d1_total / c_s / 1e9,
                                                "ms_per_step": c_s * 1e3,
                                                "api": "the bare zpir_db_answer call on host "
                                                       "limb arrays (no Python int conversion)"}}

    db_bytes_total = D0 * d1_total
    db_bytes_rank = D0 * (hi - lo)
    value = db_bytes_total / (ms / 1e3) / 1e9
    gemv_bytes = D0 * (hi - lo) + 4 * D0 + 4 * (hi - lo)
    peak, peak_src = _peaks()
    achieved = gemv_bytes / (gemv_step_ms / 1e3) / 1e9
    achieved_alone = gemv_bytes / (gemv_ms / 1e3) / 1e9
    answer_bytes = gemv_bytes + 4 * N_LWE * (hi - lo) + 256 * N_LWE + 256 * (g_hi - g_lo)
    cpu = None
    if rank == 0 and world == 1 and not args.no_cpu_baseline:
        cpu = cpu_baseline(m)
    if rank == 0:
        h2d = 4 * D0 + 4 * kctx.lm * N_LWE
        d2h = 4 * kctx.lm * params.d1_prime
        out = {
            "metric": "online server throughput (DB GB/s per query)",
            "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": max(args.warmup, 3), "ms_per_step": ms, "higher_is_better": True,
            "scaling": "weak", "vs_baseline": None, "dtype": "u8xu32 mod 2^32 / 2048-bit Montgomery",
            "data": "synthetic (seeded uniform u8 DB, uniform qu0 / ck_o, seeded Paillier modulus)",
            "config": _config(world), "parallelism": f"db-row shards x{world}",
            "gpu_launches": 6 * args.steps,   # qplanes, GEMV, build_bc, compression, groups_z, finish
            "roofline": {"bound": "hbm",
                         "kernel": "umma_gemm_kernel<16,0> (tcgen05 GEMV + query planes) inside the "
                                   "full answer step, on SMs - COMPRESS_CTAS, concurrent with the "
                                   "compression GEMM (external timing events in the step graph; mean of "
                                   "the last replay of 10 runs of 20 back-to-back steps)",
                         "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": _traffic(),
                         "peak_source": peak_src,
                         "bytes_per_launch": gemv_bytes, "ms_in_step": gemv_step_ms,
                         "alone_all_sms": {"ms": gemv_ms, "achieved": achieved_alone,
                                           "frac": achieved_alone / peak}},
            "answer_roofline": {"bytes": answer_bytes, "ms": ms,
                                "achieved_gbs": answer_bytes / (ms / 1e3) / 1e9,
                                "frac": answer_bytes / (ms / 1e3) / 1e9 / peak,
                                "gemv_ms": gemv_ms, "compress_plus_groups_ms": comp_ms,
                                "side_ms_in_step": side_step_ms,
                                "schedule": f"GEMV on {plan.sms - plan.ctas} SMs || compression on "
                                            f"{plan.ctas} SMs, then group stage; CUDA graph"},
            "e2e": {"value": db_bytes_total / e2e_s / 1e9, "unit": "GB/s",
                    "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h,
                    "ms_per_step": e2e_s * 1e3, "api": api},
            "clocks": clk,
            **extra_e2e,
            "setup_s": setup_s, "hint_s_per_client": hint_s,
            "per_gpu_db_bytes": db_bytes_rank,
        }
        if cpu is not None:
            out["cpu_baseline"] = {k: cpu[k] for k in ("value", "unit", "cores", "kind", "sample")}
        print(json.dumps(out), flush=True)
    if world > 1:
        dist.destroy_process_group()


def run_extra(args):
    """Non-default workloads (printed as one JSON line each, rank 0)."""
    import torch
    rank, world, local = _dist_env()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        import torch.distributed as dist
        dist.init_process_group("nccl", device_id=dev)
        if args.workload != "8g":
            # the other workloads are single-GPU: rank 0 measures, the rest wait
            if rank != 0:
                dist.barrier()
                dist.destroy_process_group()
                return
    import paper_2603_09190_b200 as z
    from paper_2603_09190_b200 import _lib, build as zb
    from paper_2603_09190_b200.bigint import ints_to_limbs, key_ctx
    zb.build()
    _lib.load()
    stream = torch.cuda.current_stream(dev)
    m = paillier_modulus(BITS, 2048)
    kctx = key_ctx(m, dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    peak, peak_src = _peaks()
    if args.workload == "8g":
        d = 92682
        params = z.ProtocolParams(z.LweParams(N_LWE, 1 << 32, 256, 6.4), d, d, BITS)
        from paper_2603_09190_b200.shard import ShardedServer, shard_bounds
        bounds = shard_bounds(d, params.capacity, world)
        lo, hi, _, _ = bounds[rank]
        db = np.frombuffer(np.random.default_rng(8).bytes(d * d), dtype=np.uint8).reshape(d, d)
        t0 = time.perf_counter()
        srv = ShardedServer(params, db[:, lo:hi], rank, world)
        setup = time.perf_counter() - t0
        cpu_part = (np.ascontiguousarray(db[:, :CPU_SAMPLE_ROWS])
                    if rank == 0 and not args.no_cpu_baseline else None)
        del db
        st = srv.state
        plan = st.answer_plan(kctx, kctx.lm)
        rng = np.random.default_rng(3)
        q32 = np.zeros(st.layout.ld, np.uint32)
        q32[:d] = rng.integers(0, 1 << 32, d, dtype=np.uint64)
        plan.qu.copy_(torch.from_numpy(q32.view(np.int32)).to(dev).reshape(1, -1))
        r = random.Random(4)
        plan.cko.copy_(torch.from_numpy(ints_to_limbs([r.randrange(m) for _ in range(N_LWE)],
                                                      kctx.lm).view(np.int32)).to(dev))

        def step():
            plan.run("full", stream)
            if world > 1:
                from paper_2603_09190_b200.shard import gather_groups
                with torch.cuda.stream(stream):
                    gather_groups(plan.t, bounds, rank)
        for _ in range(max(args.warmup, 3)):
            step()
        torch.cuda.synchronize()
        tb = time.perf_counter()          # sustained (power-capped) state, as the 1 GiB line
        while time.perf_counter() - tb < 1.5:
            for _ in range(10):
                step()
            torch.cuda.synchronize()
        e0, e1 = ev(), ev()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()
        e0.record(stream)
        for _ in range(args.steps):
            step()
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / args.steps
        if world > 1:
            tt = torch.tensor([ms], dtype=torch.float64, device=dev)
            dist.all_reduce(tt, op=dist.ReduceOp.MAX)
            ms = tt.item()
        out = {"workload": "BASELINE configs[2]: 8 GiB DB 92682 x 92682 u8, n=1024, 2048-bit, "
                           "rows sharded group-aligned", "n_gpus": world, "scaling": "strong",
               "metric": "online server throughput (DB GB/s per query)",
               "value": d * d / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
               "per_gpu_hbm_frac": (d * (hi - lo)) / (ms / 1e3) / 1e9 / peak, "setup_s": setup}
        if cpu_part is not None:
            # the chunked restatement of the reference's respond (d0 = 92682 is
            # past its float64 bound; ref_port.PortState chunks d0 by 32768)
            from oracle import ref, ref_port
            _threads(os.cpu_count())
            A = ref.public_matrix(b"\x00" * 16, d, N_LWE, 1 << 32)
            pst = ref_port.PortState(cpu_part, A, CAP)
            rq = np.random.default_rng(13).integers(0, 1 << 32, d, dtype=np.uint64)
            rr = random.Random(14)
            ck = [rr.randrange(m) for _ in range(N_LWE)]
            ts = []
            for _ in range(5):
                t1 = time.perf_counter()
                pst.respond_t(rq, ck, m)
                ts.append(time.perf_counter() - t1)
            out["cpu_baseline"] = {
                "value": d * CPU_SAMPLE_ROWS / min(ts) / 1e9, "unit": "GB/s",
                "cores": os.cpu_count(), "kind": "port",
                "sample": f"{CPU_SAMPLE_ROWS} of {d} DB rows x d0={d}: the reference's respond "
                          "algorithm chunked over d0 (3 float64 GEMV chunks of <= 32768 records, "
                          "summed mod 2^32; RNS matvec + Garner), best of 5"}
    elif args.workload == "batch64":
        params = z.ProtocolParams(z.LweParams(N_LWE, 1 << 32, 256, 6.4), D0, D1, BITS)
        st = z.ServerGlobalState(params, db_slice(0, D1))
        nq = 64
        rng = np.random.default_rng(5)
        q32 = np.zeros((nq, st.layout.ld), np.uint32)
        q32[:, :D0] = rng.integers(0, 1 << 32, (nq, D0), dtype=np.uint64)
        qd = torch.from_numpy(q32.view(np.int32)).to(dev)
        r = random.Random(6)
        cko = np.stack([ints_to_limbs([r.randrange(m) for _ in range(N_LWE)], kctx.lm)
                        for _ in range(nq)])
        cd = torch.from_numpy(cko.view(np.int32)).to(dev)
        ks = [kctx] * nq
        for _ in range(max(args.warmup, 3)):
            st.answer_batch_device(qd, cd, ks, kctx.lm, stream)
        torch.cuda.synchronize()
        tb = time.perf_counter()          # sustained (power-capped) state
        while time.perf_counter() - tb < 1.5:
            st.answer_batch_device(qd, cd, ks, kctx.lm, stream)
            torch.cuda.synchronize()
        steps = max(3, args.steps // 20)
        evs = [[ev(), ev(), ev()] for _ in range(steps)]
        e0, e1 = ev(), ev()
        e0.record(stream)
        for i in range(steps):
            st.answer_batch_device(qd, cd, ks, kctx.lm, stream, evs[i])
        e1.record(stream)
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1) / steps
        gemv = statistics.mean(e[0].elapsed_time(e[1]) for e in evs)
        comp = statistics.mean(e[1].elapsed_time(e[2]) for e in evs)
        ops = 2 * 64 * D0 * D1
        out = {"workload": "BASELINE configs[3]: 1 GiB DB, 64 queries per step (N = 256 byte-plane "
                           "GEMV) + 64 compressions", "n_gpus": 1,
               "metric": "online server throughput (DB GB/s per query, 64 queries)",
               "value": nq * D0 * D1 / (ms / 1e3) / 1e9, "unit": "GB/s", "ms_per_step": ms,
               "gemv_ms": gemv, "compress_ms": comp,
               "gemv_u8xu32_macs_per_s": ops / 2 / (gemv / 1e3),
               "gemv_hbm_frac": (D0 * D1) / (gemv / 1e3) / 1e9 / peak}
        # end to end through respond_batch(): 64 QueryMessages with host qu0 /
        # Python-int ck_o in, 64 ResponseMessages of Python ints out
        pk = z.PaillierPublicKey(m, m.bit_length())
        reg = z.ClientRegistration(pk, b"\x05" * 16, z.client_id_of(pk))
        reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(1)] * params.d1_prime)
        qms = [z.QueryMessage(reg.client_id, 0, z.SEPARATE,
                              [r.randrange(m) for _ in range(N_LWE)],
                              q32[i, :D0].astype(np.uint64)) for i in range(nq)]
        for _ in range(2):
            z.respond_batch(st, [reg] * nq, qms)
        te = []
        for _ in range(max(3, args.steps // 40)):
            t1 = time.perf_counter()
            z.respond_batch(st, [reg] * nq, qms)
            te.append(time.perf_counter() - t1)
        e2e_s = statistics.mean(te)
        out["e2e_ints"] = {"value": nq * D0 * D1 / e2e_s / 1e9, "unit": "GB/s",
                           "ms_per_step": e2e_s * 1e3,
                           "api": "paper_2603_09190_b200.respond_batch() (Python-int ck_o in, "
                                  "Python-int t out: CPython int conversion dominates)",
                           "h2d_bytes_per_step": nq * (4 * D0 + 4 * kctx.lm * N_LWE),
                           "d2h_bytes_per_step": nq * 4 * kctx.lm * params.d1_prime}
        # the same batch on wire fields (what PirServer's frame path holds): ck_o
        # as (n, 256) LE byte rows, qu0 as u32, t limb rows out -- no Python ints
        ckw = [np.ascontiguousarray(ints_to_limbs(q.ck_o, kctx.lm).view(np.uint8)
                                    .reshape(N_LWE, 4 * kctx.lm)) for q in qms]
        quw = [np.ascontiguousarray(q32[i, :D0]) for i in range(nq)]
        args_w = ([reg] * nq, [0] * nq, [z.SEPARATE] * nq, ckw, quw)
        for _ in range(3):
            z.respond_batch_wire(st, *args_w)
        tw = []
        for _ in range(max(5, args.steps // 10)):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            z.respond_batch_wire(st, *args_w)
            tw.append(time.perf_counter() - t1)
        ew = statistics.mean(tw)
        out["e2e"] = {"value": nq * D0 * D1 / ew / 1e9, "unit": "GB/s",
                      "ms_per_step": ew * 1e3, "ratio_to_device": ew * 1e3 / ms,
                      "api": "paper_2603_09190_b200.respond_batch_wire() (wire fields in, "
                             "limb rows out)",
                      "h2d_bytes_per_step": nq * (4 * D0 + 4 * kctx.lm * N_LWE),
                      "d2h_bytes_per_step": nq * 4 * kctx.lm * params.d1_prime}
        if not args.no_cpu_baseline:
            # the reference has no batch path: 64 sequential respond()s
            # (protocol.py:333-365), here on a row sample
            _threads(os.cpu_count())
            pst = _port_state(CPU_SAMPLE_ROWS)
            rq = np.random.default_rng(15)
            qs_cpu = [(rq.integers(0, 1 << 32, D0, dtype=np.uint64),
                       [r.randrange(m) for _ in range(N_LWE)]) for _ in range(nq)]
            pst.respond_t(*qs_cpu[0], m)
            t1 = time.perf_counter()
            for qu_c, ck_c in qs_cpu:
                pst.respond_t(qu_c, ck_c, m)
            dt = time.perf_counter() - t1
            out["cpu_baseline"] = {
                "value": nq * D0 * CPU_SAMPLE_ROWS / dt / 1e9, "unit": "GB/s",
                "cores": os.cpu_count(), "kind": "port",
                "sample": f"64 sequential respond()s (the reference's algorithm, no batch path) on "
                          f"{CPU_SAMPLE_ROWS} of {D1} DB rows x d0={D0}; {dt:.2f} s"}
    elif args.workload in ("update", "hint"):
        # BASELINE configs[4]: global H, then compressed hints for 256 client
        # keys (the hint worker's batches of 16), then (update) 1% of the DB
        # rows re-drawn from a seed, the incremental state and the refresh of
        # all 256 hints -- every client measured, nothing extrapolated
        params = z.ProtocolParams(z.LweParams(N_LWE, 1 << 32, 256, 6.4), D0, D1, BITS)
        db = db_slice(0, D1)
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        st = z.ServerGlobalState(params, db)
        setup = time.perf_counter() - t0
        nclients, batch = 256, 16
        regs = []
        for j in range(nclients):
            mj = paillier_modulus(BITS, 3000 + j)
            pk = z.PaillierPublicKey(mj, mj.bit_length())
            regs.append(z.ClientRegistration(pk, j.to_bytes(2, "little") * 8, z.client_id_of(pk)))
        keep = args.workload == "update"
        z.hints(st, [(reg, 0) for reg in regs[:batch]], keep_slots=keep)   # warm-up (pool, kernels)
        torch.cuda.synchronize()
        clocks = ClockSampler(0)
        clocks.start()
        t1 = time.perf_counter()
        hints = []
        for c0 in range(0, nclients, batch):
            hints += z.hints(st, [(reg, 0) for reg in regs[c0:c0 + batch]], keep_slots=keep)
        torch.cuda.synchronize()
        t_all = time.perf_counter() - t1
        t1 = time.perf_counter()
        z.hint(st, regs[0], 0)
        torch.cuda.synchronize()
        single = time.perf_counter() - t1
        ref_mulmods = 361620 * params.d1_prime
        per = t_all / nclients
        out = {"workload": "BASELINE configs[4]: global H = DB A (1 GiB, n=1024) + compressed hints "
                           "(521 entries, 2048-bit) for 256 client keys"
                           + (", then 1% of DB rows re-drawn + incremental state + refresh of all "
                              "256 hints" if keep else ""),
               "n_gpus": 1, "metric": "compressed hints per second (256 clients)",
               "value": nclients / t_all, "unit": "clients/s", "higher_is_better": True,
               "global_hint_s": st.hint_time, "setup_s": setup,
               "hints_256_clients_s": t_all, "hint_s_per_client": per,
               "hint_single_client_s": single,
               "schedule": f"protocol.hints in batches of {batch} clients (the hint worker's batch), "
                           "tensor-core Pippenger",
               "reference_equivalent_mulmods_per_s": ref_mulmods / per}
        if keep:
            rng = np.random.default_rng(77)
            rows = np.sort(rng.choice(D1, size=D1 // 100, replace=False))
            db2 = db.copy()
            db2[:, rows] = rng.integers(0, 256, (D0, rows.size), dtype=np.uint8)
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            st2, changed = st.updated(db2)
            torch.cuda.synchronize()
            t_state = time.perf_counter() - t1
            t1 = time.perf_counter()
            new = []
            for c0 in range(0, nclients, batch):
                new += z.refresh_hints(st2, list(zip(regs[c0:c0 + batch], hints[c0:c0 + batch])),
                                       changed)
            torch.cuda.synchronize()
            t_ref = time.perf_counter() - t1
            # spot check: two refreshed hints equal full hints on the updated state
            for i in (0, nclients - 1):
                full = z.hint(st2, regs[i], 0)
                assert [c.c for c in full.entries] == [c.c for c in new[i].entries]
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            z.ServerGlobalState(params, db2, db_version=1)
            torch.cuda.synchronize()
            full_rebuild = time.perf_counter() - t1
            out.update({"changed_rows": int(changed.size), "state_update_s": t_state,
                        "state_full_rebuild_gpu_s": full_rebuild,
                        "refresh_256_clients_s": t_ref,
                        "hint_refresh_s_per_client": t_ref / nclients,
                        "refresh_speedup": t_all / t_ref,
                        "metric": "seconds to update 1% of rows and refresh 256 hints",
                        "value": t_state + t_ref, "unit": "s", "higher_is_better": False})
        out["clocks"] = clocks.stop()
        if not args.no_cpu_baseline:
            hb = cpu_hint_baseline(db, m)
            out["cpu_baseline"] = {k: hb[k] for k in ("value", "unit", "cores", "kind", "sample")}
            out["cpu_baseline"]["clients_256_s"] = hb["clients_256_s"]
            if keep:
                rb, rs = cpu_rebuild_baseline(db)
                out["cpu_baseline_update"] = {
                    "value": rb + hb["clients_256_s"], "unit": "s", "cores": os.cpu_count(),
                    "kind": "port",
                    "sample": f"reference full rebuild (ServerGlobalState.__init__ restated: "
                              f"{rs}) = {rb:.1f} s + every hint regenerated (server.py:115-124): "
                              f"256 x {hb['value']:.1f} s (multiexp sample above)"}
    elif args.workload == "tiny":
        # BASELINE configs[0]: the reference's CPU-runnable case, end to end on
        # the device: global hint, one client's compressed hint, one answer
        # (SEPARATE and COMBINED) through the public API
        d = 1024
        params = z.ProtocolParams(z.LweParams(N_LWE, 1 << 32, 256, 6.4), d, d, BITS)
        db = np.frombuffer(np.random.default_rng(7).bytes(d * d), dtype=np.uint8).reshape(d, d)
        t1 = time.perf_counter()
        st = z.ServerGlobalState(params, db)
        setup = time.perf_counter() - t1
        pk = z.PaillierPublicKey(m, m.bit_length())
        reg = z.ClientRegistration(pk, b"\x05" * 16, z.client_id_of(pk))
        ht = []
        for _ in range(5):
            torch.cuda.synchronize()
            t1 = time.perf_counter()
            reg.hints[0] = z.hint(st, reg, 0)
            ht.append(time.perf_counter() - t1)
        r = random.Random(3)
        q = z.QueryMessage(reg.client_id, 0, z.SEPARATE, [r.randrange(m) for _ in range(N_LWE)],
                           np.random.default_rng(4).integers(0, 1 << 32, d, dtype=np.uint64))
        res = {}
        for mode in (z.SEPARATE, z.COMBINED):
            for _ in range(5):
                z.respond(st, reg, q, mode=mode)
            ts = []
            for _ in range(max(20, args.steps // 4)):
                t1 = time.perf_counter()
                z.respond(st, reg, q, mode=mode)
                ts.append(time.perf_counter() - t1)
            res[mode] = statistics.median(ts)
        out = {"workload": "BASELINE configs[0]: 1024 x 1024 u8 DB, n=1024, q=2^32, 2048-bit "
                           "Paillier; global hint + one client's hint (17 entries) + answer",
               "n_gpus": 1, "setup_s": setup, "global_hint_s": st.hint_time,
               "hint_s_per_client": statistics.median(ht),
               "respond_separate_ms": res[z.SEPARATE] * 1e3,
               "respond_combined_ms": res[z.COMBINED] * 1e3,
               "metric": "online server throughput (DB GB/s per query)",
               "value": d * d / res[z.SEPARATE] / 1e9, "unit": "GB/s",
               "note": "latency-bound: 1 MiB DB; e2e through respond() with host inputs"}
    if rank == 0:
        print(json.dumps(out), flush=True)
    if world > 1:
        if args.workload != "8g":
            dist.barrier()            # release the waiting ranks
        dist.destroy_process_group()


def main():
    args = _args()
    if args.impl == "reference":
        run_reference(args)
    elif args.workload != "1g":
        run_extra(args)
    else:
        run_b200(args)


if __name__ == "__main__":
    main()
