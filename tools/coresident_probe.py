"""Can the CUDA-core (IDP4A) GEMV and the tcgen05 compression share SMs?
Times each alone and both concurrently (two streams, all SMs each)."""
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
qd = torch.from_numpy(q32.view(np.int32)).to(dev).reshape(1, -1)
r = random.Random(2)
cko = torch.from_numpy(ints_to_limbs([r.randrange(m) for _ in range(1024)], kctx.lm).view(np.int32)).to(dev)
s = torch.cuda.current_stream(dev)
s2 = torch.cuda.Stream(dev)
b = torch.empty((1, lay.rows), dtype=torch.int32, device=dev)
ws = torch.empty(lay.ld * 4, dtype=torch.int32, device=dev)
bc = device.build_bc(cko, kctx.lm, s)
zz = torch.empty((lay.rows, kctx.lm + 4), dtype=torch.int32, device=dev)
planes = device.query_planes(qd, 16, s)


def gemv_cc(stream):
    device.gemv(st.dbt, qd, 0xFFFFFFFF, out=b, ws=ws, stream=stream)


def gemv_umma(stream, ctas=0):
    device.umma_gemv(st.dbt, planes, 1, out=b, stream=stream, ctas=ctas)


def comp(stream, ctas=0):
    device.umma_answer_rows(st.H_dev, bc, b[0], 0xFFFFFFFF, kctx.lm, out=zz, stream=stream, ctas=ctas)


def timeit(fn, reps=30):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(reps):
        fn()
    e1.record(s)
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps * 1e3


def both(g, c):
    def f():
        ev = torch.cuda.Event()
        ev.record(s)
        s2.wait_event(ev)
        c(s2)
        g(s)
        ev2 = torch.cuda.Event()
        ev2.record(s2)
        s.wait_event(ev2)
    return f


print("cuda-core gemv alone", timeit(lambda: gemv_cc(s)))
print("umma gemv alone", timeit(lambda: gemv_umma(s)))
print("compression alone (148)", timeit(lambda: comp(s)))
print("cc gemv || comp(148)", timeit(both(gemv_cc, comp)))
print("cc gemv || comp(40)", timeit(both(gemv_cc, lambda st_: comp(st_, 40))))
print("umma gemv(108) || comp(40)", timeit(both(lambda st_: gemv_umma(st_, 108), lambda st_: comp(st_, 40))))
print("sequential umma gemv + comp", timeit(lambda: (gemv_umma(s), comp(s))))
