"""GEMV alone (1 GiB, one query) on a given number of SMs: is the in-step GEMV
SM-limited or HBM/contention-limited?"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_09190_b200 as z  # noqa: E402
from paper_2603_09190_b200 import device  # noqa: E402

dev = torch.device("cuda", 0)
params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, bench.D1))
q32 = np.zeros((1, st.layout.ld), np.uint32)
q32[0, :bench.D0] = np.random.default_rng(1).integers(0, 1 << 32, bench.D0, dtype=np.uint64)
qd = torch.from_numpy(q32.view(np.int32)).to(dev)
s = torch.cuda.current_stream(dev)
planes = device.query_planes(qd, 16, s)
out = torch.empty((1, st.layout.rows), dtype=torch.int32, device=dev)
for ctas in (148, 128, 120, 112, 104, 96):
    for _ in range(20):
        device.umma_gemv(st.dbt, planes, 1, out=out, stream=s, ctas=ctas)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(200):
        device.umma_gemv(st.dbt, planes, 1, out=out, stream=s, ctas=ctas)
    e1.record(s)
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / 200
    print(f"ctas={ctas}: {ms * 1e3:.1f} us -> {1.074e9 / ms / 1e6:.0f} GB/s", flush=True)
