#!/bin/bash
# A/B: single-query H planes kept L2-resident across queries (ZPIR_H_KEEP_MB).
mkdir -p gpurun_out/one
python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/one/build.log 2>&1 || { tail gpurun_out/one/build.log; exit 1; }
for mb in 0 64 96 112 0 64 96 112; do
  ZPIR_H_KEEP_MB=$mb timeout 300 python bench.py --no-cpu-baseline --no-extra-e2e > gpurun_out/one/keep_$mb.json 2> gpurun_out/one/keep_$mb.err
  python -c "
import json; d=json.load(open('gpurun_out/one/keep_$mb.json'))
print('keep_mb=$mb', 'step %.4f'%d['ms_per_step'], 'gemv_in_step %.4f'%d['roofline']['ms_in_step'], 'side %.4f'%d['answer_roofline']['side_ms_in_step'], 'e2e %.4f'%d['e2e']['ms_per_step'], d['clocks']['sm_mhz'])"
done
