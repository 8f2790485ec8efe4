#!/bin/bash
# Round-2 evidence on one B200 (run from the repo root via gpurun): the driver's
# bench line, the reference arm on the same config, every workload line, ncu
# launch lists and full captures of the GEMV, the compression and tc_step.
set -u
OUT=gpurun_out/r02c
mkdir -p $OUT
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > $OUT/build.log 2>&1 || exit 1
timeout 900 python bench.py --steps 20 --warmup 5 > $OUT/bench.json 2> $OUT/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > $OUT/bench_reference.json 2> $OUT/bench_reference.err; echo "ref rc=$?"
rm -f $OUT/workloads.jsonl
for w in tiny batch64 8g hint update; do
  timeout 1500 python bench.py --workload $w --steps 20 --warmup 3 2>> $OUT/workloads.err | tail -1 >> $OUT/workloads.jsonl
  echo "workload $w rc=$?"
done
# launch list of the bench command (the plain run exited 0 above)
python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra-e2e --e2e-steps 2 > $OUT/small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 3 --no-cpu-baseline --no-extra-e2e --e2e-steps 2 > $OUT/ncu_launch.log 2>&1
# launch list of a 16-client hint batch (the hint worker's batch)
python tools/hint_batch_once.py > $OUT/hb.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/hint16_launches.csv \
  python tools/hint_batch_once.py > $OUT/ncu_hint_launch.log 2>&1
# full captures, one kernel each
PYTHONPATH=. python tools/profile_answer.py --plan full --reps 3 > $OUT/pa.log 2>&1 && {
  ncu --set full --import-source on --clock-control none -k regex:umma_gemm_kernel -s 2 -c 1 \
    -o $OUT/gemv -f python tools/profile_answer.py --plan full --reps 3 > $OUT/ncu_gemv.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:umma_planar -s 1 -c 1 \
    -o $OUT/compress_planar -f python tools/profile_answer.py --plan full --reps 3 > $OUT/ncu_planar.log 2>&1
}
python tools/batch_once.py > $OUT/pb.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:umma_planar_pair -s 1 -c 1 \
  -o $OUT/compress_pair_batch64 -f python tools/batch_once.py > $OUT/ncu_pair.log 2>&1
PYTHONPATH=. python tools/profile_answer.py --hint --reps 0 > $OUT/ph.log 2>&1 && \
ncu --set full --import-source on --clock-control none -k regex:tc_step_kernel -s 1 -c 1 \
  -o $OUT/tc_step -f python tools/profile_answer.py --hint --reps 0 > $OUT/ncu_tc.log 2>&1
python tools/ncu_summary.py $OUT/*.ncu-rep > $OUT/ncu_summary_table.md
python tools/launch_summary.py $OUT/hint16_launches.csv > $OUT/hint16_summary.txt
python tools/launch_summary.py $OUT/launches.csv --tail 60 > $OUT/launches_summary.txt
ls -la $OUT
