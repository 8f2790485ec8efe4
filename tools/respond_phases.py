"""Host-side phases of protocol.respond()'s fast path (SEPARATE, 1 GiB config):
qu narrowing, graph 1 launch, ck_o digit staging, graph 2 launch, wait, result
ints. Prints microseconds per phase (mean of N calls) next to respond() itself."""
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
from paper_2603_09190_b200 import device, protocol  # noqa: E402
from paper_2603_09190_b200.bigint import key_ctx  # noqa: E402

dev = torch.device("cuda", 0)
params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, bench.D1))
m = bench.paillier_modulus(2048, 2048)
pk = z.PaillierPublicKey(m, m.bit_length())
reg = z.ClientRegistration(pk, b"\x05" * 16, z.client_id_of(pk))
reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(1)] * params.d1_prime)
rng = np.random.default_rng(1)
qu = rng.integers(0, 1 << 32, bench.D0, dtype=np.uint64)
r = random.Random(2)
ck = [r.randrange(m) for _ in range(1024)]
q = z.QueryMessage(reg.client_id, 0, z.SEPARATE, ck, qu)
for _ in range(20):
    z.respond(st, reg, q)
kctx = key_ctx(m, dev)
plan = st.answer_plan(kctx, kctx.lm)
stream = torch.cuda.current_stream(dev)
conv = protocol._digit_conv()
lay = st.layout
N = 200
T = {}
tr = []
for _ in range(N):
    t = time.perf_counter()
    z.respond(st, reg, q)
    tr.append(time.perf_counter() - t)
for _ in range(N):
    ts = [time.perf_counter()]
    conv.narrow_u32(qu, plan.np_qu, lay.d0); ts.append(time.perf_counter())
    plan.launch("e2e_g1", stream); device.event_record(plan.ev_gemv, stream); ts.append(time.perf_counter())
    conv.digits_into(ck, plan.np_ckd, plan.ndig_m); ts.append(time.perf_counter())
    plan.launch("e2e_g2", plan.side); ts.append(time.perf_counter())
    plan.side.synchronize(); ts.append(time.perf_counter())
    vals = conv.ints_from_digits(plan.np_td, lay.groups, plan.ndig_m); ts.append(time.perf_counter())
    z.ResponseMessage(z.SEPARATE, 0, vals, reg.hints[0].entries); ts.append(time.perf_counter())
    for name, a, b in zip(["narrow_qu", "launch_g1", "digits_ck", "launch_g2", "wait", "ints_out",
                           "message"], ts, ts[1:]):
        T[name] = T.get(name, 0.0) + (b - a) * 1e6
print(f"respond() mean {np.mean(tr) * 1e6:.1f} us, median {np.median(tr) * 1e6:.1f} us")
for k, v in T.items():
    print(f"{k:12s} {v / N:8.1f} us")
# device-only: the two graphs back to back, event-timed
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
torch.cuda.synchronize()
e0.record(stream)
for _ in range(50):
    plan.launch("e2e_g1", stream)
    device.event_record(plan.ev_gemv, stream)
    plan.launch("e2e_g2", plan.side)
    stream.wait_stream(plan.side)
e1.record(stream)
torch.cuda.synchronize()
print(f"graphs g1+g2 back to back (device, incl. copies) {e0.elapsed_time(e1) / 50 * 1e3:.1f} us")
