#!/bin/bash
mkdir -p gpurun_out/r2g
python -c "from paper_2603_09190_b200 import build; build.build()" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
timeout 900 python -m pytest tests/test_gpu_server.py tests/test_gpu_kernels.py -q -m gpu -x -k "not paper_parameters" 2>&1 | tail -2
timeout 900 python -m pytest tests/test_gpu_fullsize.py -q -m gpu -x -k "tc_hint or update" 2>&1 | tail -2
python tools/hint_timing.py 2>&1 | tail -1
python tools/hint_batch_once.py > /dev/null 2>&1 && ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/r2g/hint16_launches.csv python tools/hint_batch_once.py > /dev/null 2>&1
python tools/launch_summary.py gpurun_out/r2g/hint16_launches.csv --tail 120 2>&1 | head -20
