#!/bin/bash
mkdir -p gpurun_out/r2e
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/r2e/build.log 2>&1 || { tail gpurun_out/r2e/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_wire.py tests/test_gpu_compress.py tests/test_gpu_compat.py tests/test_gpu_kernels.py -q -m gpu -x 2>&1 | tail -4
python tools/batch_wire_profile.py 2>&1 | head -4
