#!/bin/bash
# Tensor-core hint: launch list of one 16-client batch and the per-position timeline.
mkdir -p gpurun_out/tc2
python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/tc2/build.log 2>&1 || { tail gpurun_out/tc2/build.log; exit 1; }
python tools/hint_batch_once.py --warm 0 > /dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/tc2/hint16_launches.csv python tools/hint_batch_once.py --warm 0 > gpurun_out/tc2/ncu.log 2>&1
python tools/launch_summary.py gpurun_out/tc2/hint16_launches.csv | tee gpurun_out/tc2/hint16_summary.txt
ZPIR_NVCC_EXTRA="-DZPIR_TC_TRACE" python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
python tools/tc_trace.py 2>&1 | tail -42 | tee gpurun_out/tc2/trace.txt
