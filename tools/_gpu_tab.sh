#!/bin/bash
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
timeout 300 python -m pytest tests/test_gpu_kernels.py -q -m gpu -x -k "tensor_core" 2>&1 | tail -2
timeout 600 python tools/hint_timing.py --reps 1 2>&1 | tail -1
python tools/hint_batch_once.py --warm 0 > /dev/null 2>&1 || exit 1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file /tmp/h16.csv python tools/hint_batch_once.py --warm 0 > /tmp/ncu.log 2>&1
python tools/launch_summary.py /tmp/h16.csv | head -6
