#!/bin/bash
# One focused GPU check: build, upload A/B, protocol + fullsize tests.
mkdir -p gpurun_out/one
python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/one/build.log 2>&1 || { tail gpurun_out/one/build.log; exit 1; }
timeout 300 python tools/upload_probe.py 2>&1 | grep -v Warn | tail -10
timeout 1200 python -m pytest tests/test_gpu_protocol.py tests/test_gpu_fullsize.py -q -x -m gpu 2>&1 | tail -3
