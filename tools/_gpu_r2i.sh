#!/bin/bash
# Re-entry check: all GPU tests, smoke, bench (both arms).
mkdir -p gpurun_out/r2i
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/r2i/build.log 2>&1 || { tail gpurun_out/r2i/build.log; exit 1; }
timeout 3000 python -m pytest tests -q -x -m gpu --durations=15 2>&1 | tail -30 | tee gpurun_out/r2i/pytest.log
python __graft_entry__.py smoke 2>&1 | tail -2
timeout 600 python bench.py > gpurun_out/r2i/bench.json 2> gpurun_out/r2i/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/r2i/bench_ref.json 2> gpurun_out/r2i/bench_ref.err; echo "ref rc=$?"
python -c "import json; d=json.load(open('gpurun_out/r2i/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['clocks'])"
tail -c 600 gpurun_out/r2i/bench_ref.json
