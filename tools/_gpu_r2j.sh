#!/bin/bash
# All GPU tests + batch64 / hint workloads after the table-form tensor-core hint.
mkdir -p gpurun_out/r2j
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/r2j/build.log 2>&1 || { tail gpurun_out/r2j/build.log; exit 1; }
timeout 3000 python -m pytest tests -q -x -m gpu --durations=8 2>&1 | tail -16 | tee gpurun_out/r2j/pytest.log
python __graft_entry__.py smoke 2>&1 | tail -1
timeout 600 python bench.py --workload batch64 > gpurun_out/r2j/batch64.json 2> gpurun_out/r2j/batch64.err; echo "batch64 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2j/batch64.json')); print({k: d[k] for k in ('ms_per_step','gemv_ms','compress_ms')}, d['e2e']['ms_per_step'])"
timeout 900 python bench.py --workload hint > gpurun_out/r2j/hint.json 2> gpurun_out/r2j/hint.err; echo "hint rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2j/hint.json')); print({k: d[k] for k in ('hints_256_clients_s','hint_s_per_client','hint_single_client_s')})"
