#!/bin/bash
# Experiments on the tc_step timeline (timing only, results are wrong with the toggles).
for v in "-DZPIR_TC_FINE -DZPIR_TC_NOALU -DZPIR_TC_NOGATHER -DZPIR_TC_NOSTORE -DZPIR_TC_NOLDTM" "-DZPIR_TC_FINE"; do
ZPIR_NVCC_EXTRA="-DZPIR_TC_TRACE -DZPIR_TC_MMAUNROLL $v" python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
echo "variant: $v"
timeout 300 python tools/tc_trace.py 2>&1 | tail -1
done
