#!/bin/bash
# Round-end evidence: bench lines, reference arm, workloads, ncu launch lists and
# full captures of the answer, hint-GEMM, compression and tensor-core hint kernels.
# Run on the GPU box from the repo root.
set -u
OUT=gpurun_out/prof
mkdir -p $OUT
python -c "from paper_2603_09190_b200 import build; build.build()" > $OUT/build.log 2>&1 || exit 1
python bench.py > $OUT/bench.json 2> $OUT/bench.err
python bench.py --impl reference > $OUT/bench_reference.json 2> $OUT/bench_reference.err
rm -f $OUT/workloads.jsonl
for w in tiny batch64 8g hint update; do
  timeout 900 python bench.py --workload $w --steps 20 --warmup 3 2>> $OUT/workloads.err | tail -1 >> $OUT/workloads.jsonl
done
# launch list of the bench command (plain run exited 0 above)
python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra-e2e --e2e-steps 2 > $OUT/small.json 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $OUT/launches.csv \
  python bench.py --steps 2 --warmup 1 --no-cpu-baseline --no-extra-e2e --e2e-steps 2 > $OUT/ncu_launch.log 2>&1
# launch list of one client's hint (tensor-core Pippenger)
PYTHONPATH=. python tools/profile_answer.py --hint --reps 0 > $OUT/ph.log 2>&1 && \
ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $OUT/hint_launches.csv \
  python tools/profile_answer.py --hint --reps 0 > $OUT/ncu_hint_launch.log 2>&1
# full captures, one kernel each, of one answer plan replay
PYTHONPATH=. python tools/profile_answer.py --plan full --reps 3 > $OUT/pa.log 2>&1 && {
  ncu --set full --import-source on --clock-control none -k regex:umma_gemm_kernel -s 2 -c 1 \
    -o $OUT/gemv -f python tools/profile_answer.py --plan full --reps 3 > $OUT/ncu_gemv.log 2>&1
  ncu --set full --import-source on --clock-control none -k regex:umma_planar -s 1 -c 1 \
    -o $OUT/compress_planar -f python tools/profile_answer.py --plan full --reps 3 > $OUT/ncu_planar.log 2>&1
}
# the global hint GEMM (setup): int8 tensor-pipe utilisation
ncu --set full --import-source on --clock-control none -k regex:umma_gemm_kernel -s 0 -c 1 \
  -o $OUT/hint_gemm -f python tools/profile_answer.py --plan gemv --reps 1 > $OUT/ncu_hintgemm.log 2>&1
# the tensor-core Pippenger step (64 positions per launch) and the IMAD bucket combine
ZPIR_TC_CHUNK=64 ncu --set full --import-source on --clock-control none -k regex:tc_step_kernel -s 3 -c 1 \
  -o $OUT/tc_step -f python tools/profile_answer.py --hint --reps 0 > $OUT/ncu_tc.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:bucket_combine -s 0 -c 1 \
  -o $OUT/bucket_combine -f python tools/profile_answer.py --hint --reps 0 > $OUT/ncu_bc.log 2>&1
ls -la $OUT
