#!/bin/bash
mkdir -p gpurun_out/r2d
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/r2d/build.log 2>&1 || { tail gpurun_out/r2d/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tensor_core or tc_ or slot" 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_wire.py tests/test_gpu_server.py -q -m gpu -x 2>&1 | tail -5
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "tc_hint or update" 2>&1 | tail -5
python tools/batch_wire_profile.py 2>&1 | head -4
for S in 1 0; do ZPIR_TC_STRIP=$S timeout 600 python tools/hint_timing.py 2>&1 | tail -3; done
