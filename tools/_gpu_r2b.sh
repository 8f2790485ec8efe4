#!/bin/bash
# Round-2 focused check: compat / handle ABI / protocol tests, then the bench (C-ABI e2e).
mkdir -p gpurun_out/r2b
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/r2b/build.log 2>&1 || { tail gpurun_out/r2b/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_compat.py tests/test_gpu_db_api.py tests/test_gpu_protocol.py tests/test_gpu_parity.py tests/test_gpu_wire.py -q -m gpu -x 2>&1 | tail -15
timeout 900 python bench.py --steps 20 --warmup 5 --no-cpu-baseline > gpurun_out/r2b/bench.json 2> gpurun_out/r2b/bench.err; echo "bench rc=$?"
python -c "
import json; d=json.loads(open('gpurun_out/r2b/bench.json').read().strip().splitlines()[-1])
print(d['ms_per_step'], d['e2e']['ms_per_step'], d['e2e_c_abi'], d['clocks'])"
tail -3 gpurun_out/r2b/bench.err
