"""A/B of the 1 GiB database upload: pageable torch copy vs device.upload_bytes
(pinned stages, threaded host copies), and the setup / update calls that use it."""
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import numpy as np  # noqa: E402
import torch  # noqa: E402

from paper_2603_09190_b200 import device  # noqa: E402

dev = torch.device("cuda", 0)
stream = torch.cuda.current_stream(dev)
a = np.frombuffer(np.random.default_rng(1).bytes(32768 * 32768), np.uint8).reshape(32768, 32768)
ref = torch.from_numpy(a).to(dev)
for threads in ("0", "4", "8", "16", "0", "8"):
    device.UPLOAD_THREADS = int(threads)
    ts = []
    for _ in range(4):
        torch.cuda.synchronize()
        t = time.perf_counter()
        out = device.upload_bytes(a, dev, stream)
        torch.cuda.synchronize()
        ts.append(time.perf_counter() - t)
    assert torch.equal(out, ref)
    print(f"threads={threads}: upload 1 GiB {min(ts) * 1e3:.1f} ms (median "
          f"{sorted(ts)[len(ts) // 2] * 1e3:.1f}) = {a.nbytes / min(ts) / 1e9:.1f} GB/s", flush=True)
    del out

# the handle C ABI (zpir_db_create: staged upload + transpose + A + H)
import paper_2603_09190_b200 as z  # noqa: E402
from paper_2603_09190_b200.dbapi import DeviceDatabase  # noqa: E402

params = z.ProtocolParams(z.LweParams(1024, 1 << 32, 256, 6.4), 32768, 32768, 2048)
for _ in range(3):
    t = time.perf_counter()
    d = DeviceDatabase(params, a)
    print(f"zpir_db_create 1 GiB: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
    d.close()
t = time.perf_counter()
st = z.ServerGlobalState(params, a)
torch.cuda.synchronize()
print(f"ServerGlobalState 1 GiB: {(time.perf_counter() - t) * 1e3:.1f} ms", flush=True)
