"""Measured tcgen05 kind::i8 throughput (the compression / hint GEMM roofline).

    python tools/probe_umma.py [--json profiles/umma_i8_peak.json]
"""
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
res = {}
for nacc, n in ((1, 16), (4, 16), (1, 64), (4, 64), (1, 128), (4, 128), (1, 256), (2, 256),
                (2, 144), (2, 128)):
    iters = 20000
    ms = ctypes.c_float()
    _lib.call("zpir_probe_umma_i8", sms, iters, nacc * 1000 + n, ctypes.byref(ms))
    ops = sms * iters * 4 * 2 * 128 * n * 32
    key = f"n{n}_acc{nacc}_tops"
    res[key] = ops / (ms.value / 1e3) / 1e12
    cyc = ms.value / 1e3 * 1.965e9 / (iters * 4)
    print(f"M=128 N={n:3d} K=32, {nacc} accumulators: {res[key]:8.1f} T int8 ops/s  "
          f"({cyc:.1f} cycles/MMA at 1965 MHz)")
if "--json" in sys.argv:
    p = sys.argv[sys.argv.index("--json") + 1]
    json.dump({"what": "tcgen05.mma.cta_group::1.kind::i8, M=128, K=32, resident smem operands, "
                       "one CTA per SM", "sms": sms, **res}, open(p, "w"), indent=1)
