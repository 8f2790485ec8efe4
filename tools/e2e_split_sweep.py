"""respond() end to end (host ints in / out) vs the extra SMs the host-input graphs
give the compression side, 1 GiB config:    python tools/e2e_split_sweep.py 0 4 8 12"""
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
from paper_2603_09190_b200 import plan  # noqa: E402

params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
db = bench.db_slice(0, bench.D1)
m = bench.paillier_modulus(2048, 2048)
pk = z.PaillierPublicKey(m, m.bit_length())
rng = np.random.default_rng(5)
r = random.Random(6)
ck = [r.randrange(m) for _ in range(1024)]
qu = rng.integers(0, 1 << 32, bench.D0, dtype=np.uint64)
for extra in [int(x) for x in sys.argv[1:]] or [0, 4, 8, 12]:
    plan.E2E_EXTRA_CTAS = extra
    st = z.ServerGlobalState(params, db)          # fresh state: fresh plans
    reg = z.ClientRegistration(pk, b"\x05" * 16, z.client_id_of(pk))
    reg.hints[0] = z.ClientHint(0, 0, [z.PaillierCiphertext(1)] * params.d1_prime)
    q = z.QueryMessage(reg.client_id, 0, z.SEPARATE, ck, qu)
    for _ in range(20):
        z.respond(st, reg, q)
    best = []
    for _ in range(5):
        t0 = time.perf_counter()
        for _ in range(200):
            z.respond(st, reg, q)
        best.append((time.perf_counter() - t0) / 200)
    print(f"extra={extra}: respond() e2e {min(best) * 1e6:.1f} us best, {sorted(best)[2] * 1e6:.1f} us median",
          flush=True)
    del st
    torch.cuda.empty_cache()
