#!/bin/bash
# Tensor-core hint: per-position timeline of CTA (0,0).
mkdir -p gpurun_out/tc3
ZPIR_NVCC_EXTRA="-DZPIR_TC_TRACE" python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
timeout 300 python tools/tc_trace.py 2>&1 | tail -42 | cut -c1-200 | tee gpurun_out/tc3/trace.txt
