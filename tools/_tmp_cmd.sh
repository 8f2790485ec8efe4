python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || exit 1
for P in 0 1; do
  echo "== ZPIR_PAIR=$P"
  ZPIR_PAIR=$P timeout 120 python tools/split_probe.py 2>&1 | grep -E "comp  ctas=(148|40)|plan full ctas= (32|40|48)"
  ZPIR_PAIR=$P timeout 300 python bench.py --workload batch64 --steps 20 --warmup 3 2>/dev/null | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('batch64', {k:v for k,v in d.items() if k in ('value','ms_per_step','unit')})"
done
