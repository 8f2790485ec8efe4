#!/bin/bash
# One focused GPU check: build, the handle-ABI and protocol parity tests, one bench line.
mkdir -p gpurun_out/one
python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/one/build.log 2>&1 || { tail gpurun_out/one/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_db_api.py tests/test_gpu_protocol.py -q -x -m gpu 2>&1 | tail -3
timeout 600 python bench.py > gpurun_out/one/bench.json 2> gpurun_out/one/bench.err; echo "bench rc=$?"
python -c "import json; d=json.load(open('gpurun_out/one/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['clocks'])"
