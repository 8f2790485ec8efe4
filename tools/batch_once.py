"""A few respond_batch_wire-free device steps of the 64-query batch at the 1 GiB
config (one N = 256 GEMV + the CTA-pair planar compression), for ncu:

    ncu --set full -k regex:umma_planar_pair -s 1 -c 1 python tools/batch_once.py
"""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import torch  # noqa: E402

import bench  # noqa: E402

sys.argv = [sys.argv[0], "--workload", "batch64", "--steps", "3", "--warmup", "1",
            "--no-cpu-baseline"]
bench.main()
torch.cuda.synchronize()
