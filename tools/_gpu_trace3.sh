#!/bin/bash
ZPIR_NVCC_EXTRA="-DZPIR_TC_TRACE" python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
python tools/tc_trace.py 2>&1 | tail -2
python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tensor_core or tc_ or slot" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "tc_hint or update" 2>&1 | tail -2
python tools/hint_timing.py 2>&1 | tail -1
