#!/bin/bash
# tc_step timeline + parity + timing.
mkdir -p gpurun_out/tc5
ZPIR_NVCC_EXTRA="-DZPIR_TC_TRACE" python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
timeout 300 python tools/tc_trace.py 2>&1 | tail -42 > gpurun_out/tc5/trace.txt
head -1 gpurun_out/tc5/trace.txt; tail -5 gpurun_out/tc5/trace.txt
python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tensor_core" 2>&1 | tail -2
timeout 600 python tools/hint_timing.py 2>&1 | tail -1
