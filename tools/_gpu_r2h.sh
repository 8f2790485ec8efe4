#!/bin/bash
python -c "from paper_2603_09190_b200 import build; build.build()" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_server.py tests/test_gpu_kernels.py tests/test_gpu_db_api.py -q -m gpu -x -k "not paper_parameters" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "tc_hint or update" 2>&1 | tail -2
python tools/hint_timing.py 2>&1 | tail -1
python tools/hint_phases.py 2>&1 | tail -8
