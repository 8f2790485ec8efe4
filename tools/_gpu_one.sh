#!/bin/bash
# One focused GPU check: build, the batch parity tests, batch64 workload A/B on host threads.
mkdir -p gpurun_out/one
python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/one/build.log 2>&1 || { tail gpurun_out/one/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py -q -x -m gpu -k "batch" 2>&1 | tail -3
for t in 1 8 1 8; do
  ZPIR_HOST_THREADS=$t timeout 600 python bench.py --workload batch64 --steps 20 --warmup 3 2> gpurun_out/one/b64_$t.err | tail -1 > gpurun_out/one/b64_$t.json
  echo "threads=$t"; python -c "import json; d=json.load(open('gpurun_out/one/b64_$t.json')); print(d['ms_per_step'], d.get('e2e'))"
done
