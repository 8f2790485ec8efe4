"""Where does the answer's time go? Times (CUDA events, 1 GiB config):
GEMV alone on k SMs, compression alone on k SMs, and the overlapped plan."""
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
planes = device.query_planes(qd, 16, s)
b = torch.empty((1, lay.rows), dtype=torch.int32, device=dev)
bc = device.build_bc(cko, kctx.lm, s)
zz = torch.empty((lay.rows, kctx.lm + 4), dtype=torch.int32, device=dev)
flush = torch.empty(256 << 20, dtype=torch.uint8, device=dev)


def timeit(fn, reps=50):
    for _ in range(5):
        fn()
    torch.cuda.synchronize()
    tot = 0.0
    for _ in range(reps):
        flush.zero_()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record(s)
        fn()
        e1.record(s)
        torch.cuda.synchronize()
        tot += e0.elapsed_time(e1)
    return tot / reps * 1e3


for k in (148, 128, 118, 108, 98, 88):
    print(f"gemv  ctas={k:3d}: {timeit(lambda: device.umma_gemv(st.dbt, planes, 1, out=b, stream=s, ctas=k)):7.1f} us")
for k in (148, 74, 48, 40, 32, 24):
    print(f"comp  ctas={k:3d}: {timeit(lambda: device.umma_answer_rows(st.H_dev, bc, b[0], lay.qmask, kctx.lm, out=zz, stream=s, ctas=k)):7.1f} us")
plan = st.answer_plan(kctx, kctx.lm)
plan.qu.copy_(qd)
plan.cko.copy_(cko)
for c in (0, 24, 32, 40, 48):
    plan.ctas = c
    plan.graphs.clear()
    print(f"plan full ctas={c:3d}: {timeit(lambda: plan.run('full', s)):7.1f} us")
print(f"plan compress (all SMs, + groups): {timeit(lambda: plan.run('compress', s)):7.1f} us")
print(f"groups_z only: {timeit(lambda: plan._groups_z(s)):7.1f} us")
print(f"finish only: {timeit(lambda: plan._finish(s)):7.1f} us")
print(f"build_bc only: {timeit(lambda: device.build_bc(cko, kctx.lm, s, bc=bc)):7.1f} us")
print(f"qplanes only: {timeit(lambda: device.query_planes(qd, 16, s, planes=planes)):7.1f} us")
