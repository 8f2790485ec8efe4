"""Wall-clock breakdown of protocol.respond() phases at the 1 GiB config."""
import os, random, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np, torch
import bench
import paper_2603_09190_b200 as z
from paper_2603_09190_b200 import device, protocol
from paper_2603_09190_b200.bigint import key_ctx

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
stream = torch.cuda.current_stream(dev)
conv = protocol._digit_conv()
T = {}
def tick(name, t0):
    T[name] = T.get(name, 0.0) + (time.perf_counter() - t0) * 1e6
N = 50
for _ in range(N):
    t = time.perf_counter(); z.respond(st, reg, q); tick("respond_total", t)
    t = time.perf_counter()
    hq = plan.h_qu.numpy().view(np.uint32); np.copyto(hq[:bench.D0], qu, casting="unsafe"); tick("stage_qu", t)
    t = time.perf_counter()
    with torch.cuda.stream(stream): plan.qu.view(-1).copy_(plan.h_qu, non_blocking=True)
    tick("h2d_qu_enqueue", t)
    t = time.perf_counter(); plan.run("gemv", stream); tick("gemv_replay_enqueue", t)
    t = time.perf_counter(); conv.digits_into(ck, plan.h_ckd.numpy(), plan.ndig_m); tick("digits_into", t)
    t = time.perf_counter()
    with torch.cuda.stream(stream): plan.d_ckd.copy_(plan.h_ckd, non_blocking=True)
    tick("h2d_ck_enqueue", t)
    t = time.perf_counter(); plan.run("compress_digits", stream); tick("compress_replay_enqueue", t)
    t = time.perf_counter()
    with torch.cuda.stream(stream): plan.h_td.copy_(plan.d_td, non_blocking=True)
    tick("d2h_enqueue", t)
    t = time.perf_counter(); stream.synchronize(); tick("sync_wait", t)
    t = time.perf_counter(); conv.ints_from_digits(plan.h_td.numpy(), plan.h_td.shape[0], plan.ndig_m); tick("ints_from_digits", t)
    e0, e1, e2 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(stream); plan.run("gemv", stream); e1.record(stream); plan.run("compress_digits", stream); e2.record(stream)
    stream.synchronize()
    T["gpu_gemv"] = T.get("gpu_gemv", 0) + e0.elapsed_time(e1) * 1e3
    T["gpu_compress"] = T.get("gpu_compress", 0) + e1.elapsed_time(e2) * 1e3
for k, v in T.items():
    print(f"{k:28s} {v / N:8.1f} us")
