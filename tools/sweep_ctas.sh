#!/bin/bash
# sweep the SM split between the compression GEMM and the GEMV
for c in 0 12 16 20 24 32; do
  echo "ctas=$c $(ZPIR_COMPRESS_CTAS=$c python bench.py --steps 100 --warmup 5 --e2e-steps 20 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us gemv", round(d["answer_roofline"]["gemv_ms"]*1e3,1), "e2e", round(d["e2e"]["ms_per_step"]*1e3,1))')"
done
