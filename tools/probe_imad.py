"""Measure the device IMAD peak (32-bit mad.lo/mad.hi) -> profiles/imad_peak.json."""
import ctypes
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402
from paper_2603_09190_b200 import _lib, build  # noqa: E402

build.build()
_lib.load()
sms = torch.cuda.get_device_properties(0).multi_processor_count
best = 0.0
for occ in (4, 8):
    blocks, iters = sms * occ, 20000
    ms = ctypes.c_float()
    _lib.call("zpir_probe_imad", blocks, iters, ctypes.byref(ms))
    ops = blocks * 256 * iters * 16
    rate = ops / (ms.value / 1e3)
    best = max(best, rate)
    print(f"blocks={blocks} {ms.value:.2f} ms -> {rate / 1e12:.2f} T IMAD/s")
out = {"imad_per_s": best, "how": "imad_probe_kernel: 8 independent mad.lo/mad.hi chains per "
       "thread, 256 threads x (4|8) x #SMs blocks, CUDA events, best", "sms": sms,
       "device": torch.cuda.get_device_name(0)}
os.makedirs(os.path.join(ROOT, "gpurun_out"), exist_ok=True)
json.dump(out, open(os.path.join(ROOT, "gpurun_out", "imad_peak.json"), "w"), indent=1)
print(json.dumps(out))
