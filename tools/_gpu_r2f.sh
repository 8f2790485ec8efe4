#!/bin/bash
# full GPU suite + smoke after the round-2 kernel changes
mkdir -p gpurun_out/r2f
python -c "import __graft_entry__ as g; g.build(); g.smoke()" > gpurun_out/r2f/smoke.log 2>&1; echo "smoke rc=$?"; tail -1 gpurun_out/r2f/smoke.log
timeout 2400 python -m pytest tests -m gpu -q -x --durations=10 > gpurun_out/r2f/pytest.log 2>&1; echo "pytest rc=$?"; tail -16 gpurun_out/r2f/pytest.log
