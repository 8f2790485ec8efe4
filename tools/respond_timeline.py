"""Host/device timeline of one protocol.respond() (two-graph plan path) at the
1 GiB config: host timestamps of each step and device events relative to entry."""
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
side = plan.side
conv = protocol._digit_conv()
lay = st.layout
E = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
rows = []
for it in range(60):
    H = {}
    ev = {k: E() for k in ("start", "g1_end", "g2_end")}
    for e in ev.values():
        e.record(s)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    device.event_record(ev["start"], s)
    conv.narrow_u32(q.qu0, plan.np_qu, lay.d0)
    H["narrow"] = time.perf_counter()
    plan.launch("e2e_g1", s)
    device.event_record(plan.ev_gemv, s)
    device.event_record(ev["g1_end"], s)
    H["g1_launched"] = time.perf_counter()
    conv.digits_into(q.ck_o, plan.np_ckd, plan.ndig_m)
    H["digits"] = time.perf_counter()
    plan.launch("e2e_g2", side)
    device.event_record(ev["g2_end"], side)
    H["g2_launched"] = time.perf_counter()
    side.synchronize()
    H["synced"] = time.perf_counter()
    vals = conv.ints_from_digits(plan.np_td, lay.groups, plan.ndig_m)
    H["ints"] = time.perf_counter()
    if it >= 10:
        row = {k: (v - t0) * 1e6 for k, v in H.items()}
        row["dev_g1_end"] = ev["start"].elapsed_time(ev["g1_end"]) * 1e3
        row["dev_g2_end"] = ev["start"].elapsed_time(ev["g2_end"]) * 1e3
        rows.append(row)
for k in rows[0]:
    print(f"{k:14s} {statistics.median(x[k] for x in rows):8.1f} us")
t = []
for _ in range(50):
    a = time.perf_counter()
    z.respond(st, reg, q)
    t.append((time.perf_counter() - a) * 1e6)
print("respond() median", statistics.median(t))
