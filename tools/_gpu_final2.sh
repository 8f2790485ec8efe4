#!/bin/bash
# Closing check of the round: every GPU test, smoke, the default bench line and the reference arm.
mkdir -p gpurun_out/final5
python -c "from paper_2603_09190_b200 import build; build.build(); from oracle import c; c.build()" > gpurun_out/final5/build.log 2>&1 || { tail gpurun_out/final5/build.log; exit 1; }
timeout 3000 python -m pytest tests -q -x -m gpu 2>&1 | tail -4 | tee gpurun_out/final5/pytest.log
python __graft_entry__.py smoke 2>&1 | tail -1 | tee gpurun_out/final5/smoke.log
timeout 900 python bench.py > gpurun_out/final5/bench.json 2> gpurun_out/final5/bench.err; echo "bench rc=$?"
timeout 900 python bench.py --impl reference > gpurun_out/final5/bench_reference.json 2> gpurun_out/final5/bench_reference.err; echo "ref rc=$?"
python -c "import json; d=json.load(open('gpurun_out/final5/bench.json')); print(d['ms_per_step'], d['e2e']['ms_per_step'], d['roofline']['frac'], d['answer_roofline']['frac'], d['clocks'], d.get('hint_s_per_client'))"
python -c "import json; d=json.load(open('gpurun_out/final5/bench_reference.json')); print(d['value'], d['ms_per_step'])"
