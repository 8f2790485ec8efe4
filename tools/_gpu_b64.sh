#!/bin/bash
# Batched compression: parity of the planar pair kernel, the batch64 workload line.
mkdir -p gpurun_out/b64
python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/b64/build.log 2>&1 || { tail gpurun_out/b64/build.log; exit 1; }
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py -q -m gpu -x -k "planar or batch or pair" 2>&1 | tail -4
[ ${PIPESTATUS[0]} -eq 0 ] || exit 1
timeout 600 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "batch" 2>&1 | tail -3
for i in 1 2; do
timeout 600 python bench.py --workload batch64 > gpurun_out/b64/batch64_$i.json 2> gpurun_out/b64/batch64.err; echo "batch64 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/b64/batch64_$i.json')); print({k: d[k] for k in ('ms_per_step','gemv_ms','compress_ms')}, d['e2e']['ms_per_step'])"
done
