"""Run the 1 GiB online answer a few times (for ncu launch lists / captures).

    python tools/profile_answer.py [--reps 5] [--engine umma|cuda_core] [--hint]
"""
import argparse
import os
import random
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_09190_b200 as z  # noqa: E402
from paper_2603_09190_b200.bigint import ints_to_limbs, key_ctx  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--reps", type=int, default=5)
ap.add_argument("--engine", default="umma")
ap.add_argument("--hint", action="store_true")
ap.add_argument("--d1", type=int, default=bench.D1)
ap.add_argument("--plan", default="", help="run the captured plan: full | gemv | compress")
a = ap.parse_args()
dev = torch.device("cuda", 0)
params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, a.d1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, a.d1), engine=a.engine)
m = bench.paillier_modulus(2048, 2048)
kctx = key_ctx(m, dev)
rng = np.random.default_rng(1)
q32 = np.zeros(st.layout.ld, np.uint32)
q32[:bench.D0] = rng.integers(0, 1 << 32, bench.D0, dtype=np.uint64)
qd = torch.from_numpy(q32.view(np.int32)).to(dev).reshape(1, -1)
r = random.Random(2)
cko = torch.from_numpy(ints_to_limbs([r.randrange(m) for _ in range(1024)], kctx.lm).view(np.int32)).to(dev)
stream = torch.cuda.current_stream(dev)
if a.plan:
    plan = st.answer_plan(kctx, kctx.lm)
    plan.qu.copy_(qd)
    plan.cko.copy_(cko)
    for _ in range(a.reps):
        plan.run(a.plan, stream)
else:
    for _ in range(a.reps):
        st.answer_device(qd, cko, kctx, kctx.lm, stream)
if a.hint:
    pk = z.PaillierPublicKey(m, m.bit_length())
    reg = z.ClientRegistration(pk, b"\x05" * 16, z.client_id_of(pk))
    z.hint(st, reg, 0)
torch.cuda.synchronize()
print("ok")
