"""Which pieces of the captured answer plan cost what? (1 GiB config)
Each variant is captured into a CUDA graph and replayed back to back."""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_09190_b200 as z  # noqa: E402
from paper_2603_09190_b200 import device  # noqa: E402
from paper_2603_09190_b200.bigint import ints_to_limbs, key_ctx  # noqa: E402

dev = torch.device("cuda", 0)
params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, bench.D1))
m = bench.paillier_modulus(2048, 2048)
kctx = key_ctx(m, dev)
lay = st.layout
rng = np.random.default_rng(1)
q32 = np.zeros(lay.ld, np.uint32)
q32[:bench.D0] = rng.integers(0, 1 << 32, bench.D0, dtype=np.uint64)
r = random.Random(2)
plan = st.answer_plan(kctx, kctx.lm)
plan.qu.copy_(torch.from_numpy(q32.view(np.int32)).to(dev).reshape(1, -1))
plan.cko.copy_(torch.from_numpy(ints_to_limbs([r.randrange(m) for _ in range(1024)], kctx.lm).view(np.int32)).to(dev))
s = torch.cuda.current_stream(dev)
C = plan.ctas
S = plan.sms


def seq(flags):
    def f(stream):
        ev_in, ev_c = torch.cuda.Event(), torch.cuda.Event()
        ev_in.record(stream)
        plan.side.wait_event(ev_in)
        if "bc" in flags:
            device.build_bc(plan.cko, kctx.lm, stream=plan.side, bc=plan.bc)
        if "comp" in flags:
            device.umma_answer_rows(st.H_dev, plan.bc, plan.b[0], 0xFFFFFFFF, kctx.lm, out=plan.z,
                                    stream=plan.side, ctas=C)
        if "gz" in flags:
            plan._groups_z(plan.side)
        ev_c.record(plan.side)
        if "qp" in flags:
            device.query_planes(plan.qu, 16, stream, planes=plan.planes)
        if "gemv" in flags:
            device.umma_gemv(st.dbt, plan.planes, 1, out=plan.b, stream=stream, ctas=S - C)
        stream.wait_event(ev_c)
        if "fin" in flags:
            plan._finish(stream)
    return f


def graph_time(fn, reps=100):
    fn(s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    cap = torch.cuda.Stream(dev)
    cap.wait_stream(s)
    with torch.cuda.graph(g, stream=cap):
        fn(cap)
    s.wait_stream(cap)
    for _ in range(5):
        g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        g.replay()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


ALL = {"bc", "comp", "gz", "qp", "gemv", "fin"}
if "--burn" in sys.argv:
    import time
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 2.0:
        for _ in range(50):
            plan.run("full", s)
        torch.cuda.synchronize()
    print("after 2 s burn-in")
if "--sweep" in sys.argv:
    for c in (32, 40, 48, 56, 64):
        plan.ctas = C = c
        print(f"ctas={c}: full {graph_time(seq(ALL)):7.1f} us  side-only {graph_time(seq({'bc', 'comp', 'gz'})):7.1f}"
              f"  gemv-only {graph_time(seq({'qp', 'gemv'})):7.1f}")
    sys.exit(0)
print("full plan (plan.run)", graph_time(lambda st_: plan._seq("full", st_)))
for drop in [None, "fin", "gz", "bc", "qp", "comp", "gemv"]:
    fl = ALL - {drop} if drop else ALL
    print(f"without {drop!s:5s}: {graph_time(seq(fl)):7.1f} us")
print(f"gemv only (108): {graph_time(seq({'gemv'})):7.1f} us")
print(f"qp+gemv (108): {graph_time(seq({'qp', 'gemv'})):7.1f} us")
print(f"gemv+comp: {graph_time(seq({'gemv', 'comp'})):7.1f} us")
print(f"bc+comp+gz: {graph_time(seq({'bc', 'comp', 'gz'})):7.1f} us")
