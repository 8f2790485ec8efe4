"""Planar vs byte-shifted compression GEMM at the 1 GiB config."""
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_09190_b200 as z  # noqa: E402
from paper_2603_09190_b200 import device, protocol  # noqa: E402
from paper_2603_09190_b200.bigint import ints_to_limbs, key_ctx  # noqa: E402

dev = torch.device("cuda", 0)
params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, bench.D1))
m = bench.paillier_modulus(2048, 2048)
kctx = key_ctx(m, dev)
lay = st.layout
r = random.Random(2)
cko = torch.from_numpy(ints_to_limbs([r.randrange(m) for _ in range(1024)], kctx.lm).view(np.int32)).to(dev)
s = torch.cuda.current_stream(dev)
zz = torch.empty((lay.rows, kctx.lm + 4), dtype=torch.int32, device=dev)


def timeit(fn, reps=50):
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


ref = None
for planar in (False, True):
    protocol.PLANAR = planar
    for c in (0, 40, 32, 24):
        t = timeit(lambda: st.compress_rows(cko, kctx.lm, s, out=zz, ctas=c))
        print(f"planar={planar} ctas={c or 148}: compress {t:7.1f} us")
    out = zz.clone()
    if ref is None:
        ref = out
    else:
        print("planar == shifted:", torch.equal(ref, out))
    cd = cko.unsqueeze(0).expand(64, -1, -1).contiguous()
    print(f"planar={planar} batch 64 compress: {timeit(lambda: st.compress_rows(cd, kctx.lm, s), 5):9.1f} us")
