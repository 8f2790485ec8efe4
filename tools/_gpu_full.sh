#!/bin/bash
# Full-size parity (BASELINE configs[1]-[4]) on one B200.
mkdir -p gpurun_out/full
nproc > gpurun_out/full/nproc.txt; free -g >> gpurun_out/full/nproc.txt
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/full/build.log 2>&1 || { tail gpurun_out/full/build.log; exit 1; }
timeout 2400 python -m pytest tests/test_gpu_fullsize.py -q -x -m gpu --durations=0 2>&1 | tail -40 | tee gpurun_out/full/pytest.log
