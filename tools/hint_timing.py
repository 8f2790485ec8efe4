"""Per-client hint time at the 1 GiB config: one client alone and a batch of
clients through protocol.hints (the hint worker's batch), wall clock around
synchronised calls after a warm-up; entries checked equal across runs.

    python tools/hint_timing.py [--batch 16] [--reps 2]
"""
import argparse
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_09190_b200 as z  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--reps", type=int, default=2)
a = ap.parse_args()
params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, bench.D1))
regs = []
for j in range(a.batch):
    mj = bench.paillier_modulus(2048, 3000 + j)
    pk = z.PaillierPublicKey(mj, mj.bit_length())
    regs.append(z.ClientRegistration(pk, bytes([j]) * 16, z.client_id_of(pk)))
ref = z.hints(st, [(r, 0) for r in regs])            # warm-up + reference entries
torch.cuda.synchronize()
t1s, tbs = [], []
for _ in range(a.reps):
    t = time.perf_counter()
    h = z.hint(st, regs[0], 0)
    torch.cuda.synchronize()
    t1s.append(time.perf_counter() - t)
    assert [c.c for c in h.entries] == [c.c for c in ref[0].entries]
    t = time.perf_counter()
    hs = z.hints(st, [(r, 0) for r in regs])
    torch.cuda.synchronize()
    tbs.append((time.perf_counter() - t) / a.batch)
    assert all([c.c for c in x.entries] == [c.c for c in y.entries] for x, y in zip(hs, ref))
print(f"single {min(t1s):.4f} s, batched {a.batch}: {min(tbs):.4f} s per client")
