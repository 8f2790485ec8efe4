"""Timeline of tc_step for CTA (0, 0): build the library with -DZPIR_TC_TRACE
(on the GPU box only: ZPIR_NVCC_EXTRA=-DZPIR_TC_TRACE), run one client's hint,
print per-position stage times (cycles relative to the position start).

    ZPIR_NVCC_EXTRA=-DZPIR_TC_TRACE python -c "from paper_2603_09190_b200 import build; build.build(force=True)"
    python tools/tc_trace.py
"""
import ctypes
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_09190_b200 as z  # noqa: E402
from paper_2603_09190_b200 import _lib  # noqa: E402

params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, bench.D1))
m = bench.paillier_modulus(2048, 2048)
pk = z.PaillierPublicKey(m, m.bit_length())
reg = z.ClientRegistration(pk, b"\x05" * 16, z.client_id_of(pk))
z.hint(st, reg, 0)
torch.cuda.synchronize()
buf = (ctypes.c_ulonglong * (64 * 16))()
rc = _lib.lib().zpir_tc_trace(buf)
assert rc == 0
t = np.array(buf, dtype=np.int64).reshape(64, 16)
names = ["start", "Ardy", "Adrn", "-", "gissue", "Brdy", "Bdrn", "publ", "-", "-",
         "-", "m:XA", "m:XB", "m:Xend", "m:Yend", "Bwait"]
print("pos " + " ".join(f"{n:>7s}" for n in names) + "  period")
for p in range(1, 40):
    rel = t[p] - t[p, 0]
    rel[15] = t[p, 15]          # cumulative B-tile wait of the MMA thread (cycles)
    per = t[p + 1, 0] - t[p, 0] if p + 1 < 64 else 0
    print(f"{p:3d} " + " ".join(f"{int(x):7d}" for x in rel) + f"  {int(per):7d}")
rows = []
for p in range(2, 60):
    rr = t[p] - t[p, 0]
    rr[15] = t[p, 15]
    rows.append(rr)
med = np.median(np.stack(rows), axis=0)
print("med " + " ".join(f"{int(x):7d}" for x in med) + f"  {int(np.median(np.diff(t[2:60, 0]))):7d}")
