"""Host/device timeline of one protocol.respond() (plan path) at the 1 GiB config:
host timestamps of each step and device event times relative to the call entry."""
import os
import random
import statistics
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
for _ in range(5):
    z.respond(st, reg, q)
kctx = key_ctx(m, dev)
plan = st.answer_plan(kctx, kctx.lm)
s = torch.cuda.current_stream(dev)
conv = protocol._digit_conv()
lay = st.layout
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
rows = []
for it in range(40):
    H = {}
    ev = {k: E() for k in ("start", "qu_in", "gemv_end", "side_end", "finish_end", "out")}
    t0 = time.perf_counter()
    ev["start"].record(s)
    hq = plan.h_qu.numpy().view(np.uint32)
    np.copyto(hq[: lay.d0], q.qu0, casting="unsafe")
    H["stage_qu"] = time.perf_counter()
    device.h2d_async(plan.qu, plan.h_qu, s)
    ev["qu_in"].record(s)
    plan.ev_in.record(s)
    plan.run("gemv_part", s)
    ev["gemv_end"].record(s)
    H["gemv_launched"] = time.perf_counter()
    conv.digits_into(q.ck_o, plan.h_ckd.numpy(), plan.ndig_m)
    H["digits"] = time.perf_counter()
    side = plan.side
    side.wait_event(plan.ev_in)
    device.h2d_async(plan.d_ckd, plan.h_ckd, side)
    plan.run("side_digits", side)
    ev["side_end"].record(side)
    s.wait_stream(side)
    plan.run("finish_digits", s)
    ev["finish_end"].record(s)
    device.d2h_async(plan.h_td, plan.d_td, s)
    ev["out"].record(s)
    H["all_launched"] = time.perf_counter()
    s.synchronize()
    H["synced"] = time.perf_counter()
    vals = conv.ints_from_digits(plan.h_td.numpy(), plan.h_td.shape[0], plan.ndig_m)
    H["ints"] = time.perf_counter()
    if it >= 5:
        row = {k: (v - t0) * 1e6 for k, v in H.items()}
        for k in ("qu_in", "gemv_end", "side_end", "finish_end", "out"):
            row["dev_" + k] = ev["start"].elapsed_time(ev[k]) * 1e3
        rows.append(row)
for k in rows[0]:
    print(f"{k:18s} {statistics.median(r[k] for r in rows):8.1f} us")
t = []
for _ in range(30):
    a = time.perf_counter()
    z.respond(st, reg, q)
    t.append((time.perf_counter() - a) * 1e6)
print("respond() median", statistics.median(t))
