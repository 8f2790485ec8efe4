#!/bin/bash
# One focused GPU check: build, upload A/B, protocol tests, update workload.
mkdir -p gpurun_out/one
python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/one/build.log 2>&1 || { tail gpurun_out/one/build.log; exit 1; }
timeout 300 python tools/upload_probe.py 2>&1 | tail -8
timeout 900 python -m pytest tests/test_gpu_protocol.py tests/test_gpu_parity.py -q -x -m gpu 2>&1 | tail -3
timeout 600 python bench.py --workload update --steps 20 --warmup 3 2> gpurun_out/one/upd.err | tail -1 > gpurun_out/one/upd.json; cut -c1-400 gpurun_out/one/upd.json
