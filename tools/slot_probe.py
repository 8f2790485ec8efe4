"""A/B of slot_combine (one client, 1 GiB layout: 521 groups x 63 slots, 4096-bit
m^2): kernel time by CUDA events, output bytes compared across runs."""
import hashlib
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
from paper_2603_09190_b200 import device  # noqa: E402
from paper_2603_09190_b200.bigint import ints_to_limbs, key_ctx  # noqa: E402

dev = torch.device("cuda", 0)
device.require_cuda(dev)
m = bench.paillier_modulus(2048, 2048)
kctx = key_ctx(m, dev)
groups, cap = 521, 63
rng = np.random.default_rng(9)
vals = [int.from_bytes(rng.bytes(510), "little") % (m * m) for _ in range(groups * cap)]
W = torch.from_numpy(ints_to_limbs(vals, kctx.l2).view(np.int32)).to(dev)
out = torch.empty((groups, kctx.l2), dtype=torch.int32, device=dev)
stream = torch.cuda.current_stream(dev)
device.slot_combine(W, cap, None, groups, kctx, out, 1 << 32, stream)
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(5):
    e0.record(stream)
    device.slot_combine(W, cap, None, groups, kctx, out, 1 << 32, stream)
    e1.record(stream)
    torch.cuda.synchronize()
    ts.append(e0.elapsed_time(e1))
h = hashlib.sha256(out.cpu().numpy().tobytes()).hexdigest()[:16]
print(f"ZPIR_SLOT_UNROLL={os.environ.get('ZPIR_SLOT_UNROLL', 'default (1)')} slot_combine {min(ts):.2f} ms "
      f"(median {sorted(ts)[2]:.2f}) out {h}")
