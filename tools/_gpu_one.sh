#!/bin/bash
# A/B: L2 prefetch distance of the stream-K GEMV producer (ZPIR_GEMV_PF units ahead).
mkdir -p gpurun_out/one
python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/one/build.log 2>&1 || { tail gpurun_out/one/build.log; exit 1; }
for pf in 0 8 16 32 64 0 16 32; do
  ZPIR_GEMV_PF=$pf timeout 300 python bench.py --no-cpu-baseline --no-extra-e2e > gpurun_out/one/pf_$pf.json 2> gpurun_out/one/pf_$pf.err
  python -c "
import json; d=json.load(open('gpurun_out/one/pf_$pf.json'))
print('pf=$pf', 'step %.4f'%d['ms_per_step'], 'gemv_in_step %.4f'%d['roofline']['ms_in_step'], 'alone %.4f'%d['roofline']['alone_all_sms']['ms'], 'side %.4f'%d['answer_roofline']['side_ms_in_step'], 'e2e %.4f'%d['e2e']['ms_per_step'], d['clocks']['sm_mhz'])" || tail -3 gpurun_out/one/pf_$pf.err
done
ZPIR_GEMV_PF=32 timeout 600 python -m pytest tests/test_gpu_kernels.py -q -x -m gpu -k "gemv" 2>&1 | tail -2
