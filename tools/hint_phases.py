"""Where a 16-client protocol.hints batch spends its time (1 GiB config):
every device-module call inside hints() is bracketed by CUDA events on the
caller's stream (device time) and by the host clock (wall), after a warm-up."""
import collections
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402
import paper_2603_09190_b200 as z  # noqa: E402
from paper_2603_09190_b200 import device, protocol  # noqa: E402

params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), bench.D0, bench.D1, 2048)
st = z.ServerGlobalState(params, bench.db_slice(0, bench.D1))
regs = []
for j in range(16):
    mj = bench.paillier_modulus(2048, 3000 + j)
    pk = z.PaillierPublicKey(mj, mj.bit_length())
    regs.append(z.ClientRegistration(pk, bytes([j]) * 16, z.client_id_of(pk)))
z.hints(st, [(r, 0) for r in regs])
torch.cuda.synchronize()
rec = collections.defaultdict(list)


def wrap(mod, name):
    f = getattr(mod, name)

    def g(*a, **k):
        s = torch.cuda.current_stream()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        t0 = time.perf_counter()
        e0.record(s)
        r = f(*a, **k)
        e1.record(s)
        rec[name].append((e0, e1, time.perf_counter() - t0))
        return r
    setattr(mod, name, g)


for n in ("chacha_below", "pow8_table", "slot_fixed_tc_many", "slot_combine_many"):
    wrap(device, n)
wrap(protocol, "_d2h_u32")
wrap(protocol, "key_ctx")
torch.cuda.synchronize()
start = torch.cuda.Event(enable_timing=True)
start.record(torch.cuda.current_stream())
t0 = time.perf_counter()
z.hints(st, [(r, 0) for r in regs])
torch.cuda.synchronize()
wall = time.perf_counter() - t0
print(f"hints(16): {wall:.3f} s wall, {wall / 16:.4f} s per client")
for name, v in rec.items():
    dev = sum(e0.elapsed_time(e1) for e0, e1, _ in v)
    host = sum(h for _, _, h in v)
    first = start.elapsed_time(v[0][0])
    last = start.elapsed_time(v[-1][1])
    print(f"{name:22s} calls {len(v):3d} device(stream) {dev:9.1f} ms  host {1e3 * host:9.1f} ms"
          f"  span {first:8.1f} .. {last:8.1f} ms after start")
