#!/bin/bash
# Tensor-core hint: parity (vs IMAD, GMP oracle), timing, then the per-position timeline.
mkdir -p gpurun_out/tc4
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/tc4/build.log 2>&1 || { tail gpurun_out/tc4/build.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tensor_core" 2>&1 | tail -5
[ ${PIPESTATUS[0]} -eq 0 ] || exit 1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "tc_hint" 2>&1 | tail -3
timeout 600 python tools/hint_timing.py 2>&1 | tail -1
timeout 600 python tools/hint_phases.py 2>&1 | grep -E "slot_fixed_tc_many|slot_combine|hints\("
ZPIR_NVCC_EXTRA="-DZPIR_TC_TRACE" python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
timeout 300 python tools/tc_trace.py 2>&1 | tail -42 > gpurun_out/tc4/trace.txt
awk '{print $1,$2,$3,$4,$5,$6,$7,$8,$9,$13,$14,$15,$16,$17,$18}' gpurun_out/tc4/trace.txt | tail -12
