#!/bin/bash
mkdir -p gpurun_out/r2c
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/r2c/build.log 2>&1 || { tail gpurun_out/r2c/build.log; exit 1; }
timeout 1200 python -m pytest tests/test_gpu_compat.py tests/test_gpu_db_api.py tests/test_gpu_wire.py tests/test_gpu_protocol.py -q -m gpu -x 2>&1 | tail -15
timeout 900 python bench.py --workload batch64 --steps 100 --warmup 5 --no-cpu-baseline > gpurun_out/r2c/batch64.json 2> gpurun_out/r2c/batch64.err; echo "batch rc=$?"
tail -c 1500 gpurun_out/r2c/batch64.json; tail -3 gpurun_out/r2c/batch64.err
