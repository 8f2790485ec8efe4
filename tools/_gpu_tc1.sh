#!/bin/bash
# Tensor-core hint: parity of the table form (vs IMAD, vs the GMP oracle) and timing.
mkdir -p gpurun_out/tc1
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/tc1/build.log 2>&1 || { tail gpurun_out/tc1/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tensor_core" 2>&1 | tail -15
[ ${PIPESTATUS[0]} -eq 0 ] || exit 1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "tc_hint" 2>&1 | tail -5
timeout 600 python tools/hint_timing.py 2>&1 | tail -3
timeout 600 python tools/hint_phases.py 2>&1 | tail -12
