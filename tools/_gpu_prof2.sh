#!/bin/bash
# ncu --set full of the batched compression kernel and of tc_step (after plain runs exited 0).
OUT=gpurun_out/prof2
mkdir -p $OUT
python -c "from paper_2603_09190_b200 import build; build.build()" > $OUT/build.log 2>&1 || exit 1
python tools/batch_once.py > $OUT/b.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:umma_planar_pair -s 1 -c 1 \
  -o $OUT/compress_pair -f python tools/batch_once.py > $OUT/ncu_pair.log 2>&1
PYTHONPATH=. python tools/profile_answer.py --hint --reps 0 > $OUT/ph.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tc_step_kernel -s 2 -c 1 \
  -o $OUT/tc_step -f python tools/profile_answer.py --hint --reps 0 > $OUT/ncu_tc.log 2>&1
python tools/ncu_summary.py $OUT/*.ncu-rep | tee $OUT/summary.md
