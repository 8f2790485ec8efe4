"""respond_batch_wire(64) at the 1 GiB config: host staging vs device vs whole call,
plus a cProfile of the call (host hot spots)."""
import cProfile
import os
import pstats
import random
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_09190_b200 as z  # noqa: E402
from paper_2603_09190_b200 import protocol  # noqa: E402
from paper_2603_09190_b200.bigint import ints_to_limbs, key_ctx  # noqa: E402

params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, bench.D1))
m = bench.paillier_modulus(2048, 2048)
pk = z.PaillierPublicKey(m, m.bit_length())
reg = z.ClientRegistration(pk, b"\x05" * 16, z.client_id_of(pk))
reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(1)] * params.d1_prime)
rng = np.random.default_rng(5)
r = random.Random(6)
nq = 64
kc = key_ctx(m, st.device)
cks = [np.ascontiguousarray(ints_to_limbs([r.randrange(m) for _ in range(1024)], 64)
                            .view(np.uint8).reshape(1024, 256)) for _ in range(nq)]
qus = [rng.integers(0, 1 << 32, bench.D0, dtype=np.uint64).astype(np.uint32) for _ in range(nq)]
args = ([reg] * nq, [0] * nq, [z.SEPARATE] * nq, cks, qus)
for sub in (16, 32, 64, 32):
    protocol.WIRE_BATCH_SUB = sub
    for _ in range(3):
        z.respond_batch_wire(st, *args)
    torch.cuda.synchronize()
    ts = []
    for _ in range(10):
        t = time.perf_counter()
        z.respond_batch_wire(st, *args)
        ts.append(time.perf_counter() - t)
    print(f"respond_batch_wire(64), sub-batches of {sub}: {1e3 * min(ts):.2f} ms best, "
          f"{1e3 * np.median(ts):.2f} median")
B = protocol._wire_bufs.bufs
qn = B["q"].numpy().view(np.uint32)
cn = B["c"].numpy()
conv = protocol._conv_module()
t = time.perf_counter()
conv.stage_rows(qus, qn, qn.shape[1] * 4, 1, qn.shape[1] * 4, 8, True)
t1 = time.perf_counter()
conv.stage_rows(cks, cn, 1024 * 256, 1024, 256, 8, False)
t2 = time.perf_counter()
print(f"staging qu {1e3 * (t1 - t):.2f} ms, ck {1e3 * (t2 - t1):.2f} ms")
# device only
qd = B["qd"]
cd = B["cd"]
s = torch.cuda.current_stream()
ev = [torch.cuda.Event(enable_timing=True) for _ in range(2)]
for _ in range(3):
    st.answer_batch_device(qd, cd, [kc] * nq, 64, s)
ev[0].record(s)
for _ in range(10):
    st.answer_batch_device(qd, cd, [kc] * nq, 64, s)
ev[1].record(s)
torch.cuda.synchronize()
print(f"device answer_batch_device(64): {ev[0].elapsed_time(ev[1]) / 10:.2f} ms")
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    z.respond_batch_wire(st, *args)
pr.disable()
pstats.Stats(pr).sort_stats("cumulative").print_stats(25)
