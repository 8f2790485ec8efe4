#!/bin/bash
# sweep the SM split between the compression side stream and the GEMV
for c in ${@:-40 44 48 52 56 64}; do
  echo "ctas=$c $(ZPIR_COMPRESS_CTAS=$c python bench.py --steps 200 --warmup 10 --e2e-steps 5 --no-cpu-baseline 2>/dev/null | python -c 'import json,sys; d=json.loads(sys.stdin.read()); print(round(d["value"],1), round(d["ms_per_step"]*1e3,1), "us")')"
done
