#!/bin/bash
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
timeout 600 python tools/hint_timing.py --reps 2 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_server.py tests/test_gpu_fullsize.py -q -m gpu -x -k "hint or refresh or update" 2>&1 | tail -2
timeout 900 python bench.py --workload hint > /tmp/hint.json 2>/tmp/hint.err; python -c "import json; d=json.load(open('/tmp/hint.json')); print({k: d[k] for k in ('hints_256_clients_s','hint_s_per_client','hint_single_client_s')})"
