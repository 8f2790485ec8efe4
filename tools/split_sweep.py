"""Answer-step time vs the compression / GEMV SM split, 1 GiB config,
device-resident plan replays:    python tools/split_sweep.py 30 34 36 38"""
import os
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_09190_b200 as z  # noqa: E402
from paper_2603_09190_b200.bigint import ints_to_limbs, key_ctx  # noqa: E402
from paper_2603_09190_b200.plan import AnswerPlan  # noqa: E402

dev = torch.device("cuda", 0)
params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, bench.D1))
m = bench.paillier_modulus(2048, 2048)
kctx = key_ctx(m, dev)
rng = np.random.default_rng(1)
q32 = np.zeros(st.layout.ld, np.uint32)
q32[:bench.D0] = rng.integers(0, 1 << 32, bench.D0, dtype=np.uint64)
r = random.Random(2)
ck = ints_to_limbs([r.randrange(m) for _ in range(1024)], kctx.lm)
s = torch.cuda.current_stream(dev)
ref = None
for ctas in [int(x) for x in sys.argv[1:]] or [20, 24, 28, 32, 36]:
    p = AnswerPlan(st, kctx, kctx.lm, ctas)
    p.qu.copy_(torch.from_numpy(q32.view(np.int32)).to(dev).reshape(1, -1))
    p.cko.copy_(torch.from_numpy(ck.view(np.int32)).to(dev))
    for _ in range(5):
        p.run("full", s)
    torch.cuda.synchronize()
    tb = time.perf_counter()
    while time.perf_counter() - tb < 1.0:
        for _ in range(50):
            p.run("full", s)
        torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(s)
    for _ in range(200):
        p.run("full", s)
    e1.record(s)
    torch.cuda.synchronize()
    t = p.t.cpu()
    if ref is None:
        ref = t
    ok = torch.equal(ref, t)
    print(f"ctas={ctas}: {e0.elapsed_time(e1) / 200 * 1e3:.1f} us/step  same_t={ok}", flush=True)
