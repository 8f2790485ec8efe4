python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || exit 1
for T in 0 1; do
  echo "== ZPIR_TPC_PACK=$T"
  ZPIR_TPC_PACK=$T timeout 120 python tools/split_probe.py 2>&1 | grep -E "gemv  ctas=(108|118)|plan full"
  ZPIR_TPC_PACK=$T python bench.py --no-cpu-baseline --no-extra-e2e 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('bench', d['value'], d['ms_per_step'], d['e2e']['ms_per_step'])"
done
