"""One protocol.hints call for a batch of clients at the 1 GiB config (after a
warm-up batch): the launch list of the hint worker's batch under ncu.

    ncu --metrics gpu__time_duration.sum --csv python tools/hint_batch_once.py [--batch 16]
"""
import argparse
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_09190_b200 as z  # noqa: E402

ap = argparse.ArgumentParser()
ap.add_argument("--batch", type=int, default=16)
ap.add_argument("--warm", type=int, default=1)
a = ap.parse_args()
params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, bench.D1))
regs = []
for j in range(a.batch):
    mj = bench.paillier_modulus(2048, 3000 + j)
    pk = z.PaillierPublicKey(mj, mj.bit_length())
    regs.append(z.ClientRegistration(pk, bytes([j]) * 16, z.client_id_of(pk)))
for _ in range(a.warm):
    z.hints(st, [(r, 0) for r in regs])
torch.cuda.synchronize()
z.hints(st, [(r, 0) for r in regs])
torch.cuda.synchronize()
print("ok")
