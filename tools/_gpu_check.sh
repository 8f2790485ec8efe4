#!/bin/bash
# Re-entry check on the GPU box: build, smoke, parity suite, default bench line.
mkdir -p gpurun_out/chk
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/chk/smoke.log 2>&1; echo "smoke rc=$?"
timeout 1500 python -m pytest tests -q -x -m gpu > gpurun_out/chk/gpu_tests.log 2>&1; echo "tests rc=$?"; tail -5 gpurun_out/chk/gpu_tests.log
timeout 600 python bench.py > gpurun_out/chk/bench.json 2> gpurun_out/chk/bench.err; echo "bench rc=$?"; cat gpurun_out/chk/bench.json
