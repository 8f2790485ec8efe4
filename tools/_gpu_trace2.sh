#!/bin/bash
for X in 0 1 2; do
ZPIR_NVCC_EXTRA="-DZPIR_TC_TRACE -DZPIR_TC_EXP=$X" python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
echo "EXP=$X"; python tools/tc_trace.py 2>&1 | tail -2
done
