#!/bin/bash
# ncu full capture of one tc_step launch (1024 positions, 257 row tiles) with source lines
mkdir -p gpurun_out/tcprof
python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/tcprof/build.log 2>&1 || exit 1
PYTHONPATH=. python tools/profile_answer.py --hint --reps 0 > gpurun_out/tcprof/ph.log 2>&1 || { tail gpurun_out/tcprof/ph.log; exit 1; }
timeout 900 ncu --set full --import-source on --clock-control none -k regex:tc_step_kernel -s 2 -c 1 \
  -o gpurun_out/tcprof/tc_step -f python tools/profile_answer.py --hint --reps 0 > gpurun_out/tcprof/ncu.log 2>&1
echo "ncu rc=$?"; tail -3 gpurun_out/tcprof/ncu.log; ls -la gpurun_out/tcprof
