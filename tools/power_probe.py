"""Board power and SM clock while looping each piece of the answer (2 s each)."""
import os
import random
import subprocess
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_09190_b200 as z  # noqa: E402
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
for w in ("full", "gemv", "compress"):
    plan.run(w, s)
torch.cuda.synchronize()


def loop(which, secs=2.5):
    smi = subprocess.Popen(["nvidia-smi", "-i", "0", "--query-gpu=power.draw,clocks.sm",
                            "--format=csv,noheader,nounits", "-lms", "100"],
                           stdout=subprocess.PIPE, text=True)
    t0 = time.perf_counter()
    n = 0
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    while time.perf_counter() - t0 < secs:
        if n == 200:
            e0.record(s)
        for _ in range(50):
            plan.run(which, s)
        n += 50
        torch.cuda.synchronize()
    e1.record(s)
    torch.cuda.synchronize()
    smi.terminate()
    out = smi.communicate()[0].strip().splitlines()
    vals = [tuple(float(x) for x in l.split(",")) for l in out if l.count(",") == 1]
    vals = vals[len(vals) // 3:]
    pw = sorted(v[0] for v in vals)[len(vals) // 2] if vals else 0
    ck = sorted(v[1] for v in vals)[len(vals) // 2] if vals else 0
    ms = e0.elapsed_time(e1) / (n - 200)
    print(f"{which:9s}: {ms * 1e3:7.1f} us/step  power {pw:6.1f} W  sm clock {ck:6.0f} MHz")
    time.sleep(1.0)


for w in ("gemv", "compress", "full", "gemv"):
    loop(w)
