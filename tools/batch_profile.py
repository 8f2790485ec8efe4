"""cProfile of respond_batch(64) at the 1 GiB config (host-side hot spots)."""
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

params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, bench.D1))
m = bench.paillier_modulus(2048, 2048)
pk = z.PaillierPublicKey(m, m.bit_length())
reg = z.ClientRegistration(pk, b"\x05" * 16, z.client_id_of(pk))
reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(1)] * params.d1_prime)
rng = np.random.default_rng(5)
r = random.Random(6)
qms = [z.QueryMessage(reg.client_id, 0, z.SEPARATE, [r.randrange(m) for _ in range(1024)],
                      rng.integers(0, 1 << 32, bench.D0, dtype=np.uint64)) for _ in range(64)]
for _ in range(3):
    z.respond_batch(st, [reg] * 64, qms)
torch.cuda.synchronize()
t = time.perf_counter()
for _ in range(5):
    z.respond_batch(st, [reg] * 64, qms)
print("respond_batch(64) ms", (time.perf_counter() - t) / 5 * 1e3)
pr = cProfile.Profile()
pr.enable()
for _ in range(5):
    z.respond_batch(st, [reg] * 64, qms)
pr.disable()
pstats.Stats(pr).sort_stats("tottime").print_stats(14)
