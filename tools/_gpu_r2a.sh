#!/bin/bash
# Round-2 check: all GPU tests, the default bench line, the reference arm, a 2-rank gloo bench code-path run.
mkdir -p gpurun_out/r2a
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/r2a/build.log 2>&1 || { tail gpurun_out/r2a/build.log; exit 1; }
timeout 2400 python -m pytest tests -q -m gpu -x --durations=15 > gpurun_out/r2a/pytest.log 2>&1; echo "pytest rc=$?"; tail -25 gpurun_out/r2a/pytest.log
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/r2a/bench.json 2> gpurun_out/r2a/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/r2a/bench_ref.json 2> gpurun_out/r2a/bench_ref.err; echo "ref rc=$?"
timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --steps 5 --warmup 3 --dist-backend gloo --no-extra-e2e --e2e-steps 5 > gpurun_out/r2a/bench_2rank_gloo.json 2> gpurun_out/r2a/bench_2rank_gloo.err; echo "2rank rc=$?"
tail -c 600 gpurun_out/r2a/bench.json; tail -c 400 gpurun_out/r2a/bench_ref.json; tail -c 300 gpurun_out/r2a/bench_2rank_gloo.json; tail -5 gpurun_out/r2a/bench_2rank_gloo.err
