#!/bin/bash
# Digits per exponent word: hint time per client for D = 5, 6, 7, 8.
for d in 6 7 8 5; do
ZPIR_NVCC_EXTRA="-DZPIR_TC_D=$d" python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
echo "D=$d"
timeout 600 python tools/hint_timing.py --reps 1 2>&1 | tail -1
timeout 600 python tools/hint_phases.py 2>&1 | grep -E "slot_fixed_tc_many|slot_combine"
done
python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1
