#!/bin/bash
# Closing check of the round: every GPU test, smoke, then the evidence script.
mkdir -p gpurun_out/final2
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/final2/build.log 2>&1 || { tail gpurun_out/final2/build.log; exit 1; }
timeout 3000 python -m pytest tests -q -x -m gpu 2>&1 | tail -4 | tee gpurun_out/final2/pytest.log
python __graft_entry__.py smoke 2>&1 | tail -1 | tee gpurun_out/final2/smoke.log
bash tools/profile_r02.sh > gpurun_out/final2/profile.log 2>&1
tail -3 gpurun_out/final2/profile.log
