#!/bin/bash
# Refresh through the cost model: parity tests, then the update workload line.
mkdir -p gpurun_out/upd
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/upd/build.log 2>&1 || { tail gpurun_out/upd/build.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_server.py tests/test_gpu_fullsize.py -q -m gpu -x -k "refresh or update" 2>&1 | tail -3
timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_protocol.py -q -m gpu -x -k "batch" 2>&1 | tail -2
timeout 900 python bench.py --workload update > gpurun_out/upd/update.json 2> gpurun_out/upd/update.err; echo "update rc=$?"
python -c "import json; d=json.load(open('gpurun_out/upd/update.json')); print({k: d[k] for k in ('value','state_update_s','refresh_256_clients_s','hint_refresh_s_per_client','hint_s_per_client')})"
timeout 600 python bench.py --workload batch64 > gpurun_out/upd/batch64.json 2> gpurun_out/upd/batch64.err; echo "batch64 rc=$?"
python -c "import json; d=json.load(open('gpurun_out/upd/batch64.json')); print({k: d[k] for k in ('ms_per_step','gemv_ms','compress_ms')}, d['e2e']['ms_per_step'])"
