for i in 1 2; do
timeout 300 python bench.py --workload hint --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hint', d['hint_s_per_client'], d['reference_equivalent_mulmods_per_s'])"
done
ZPIR_TC_CHUNK=64 timeout 300 python bench.py --workload hint --steps 20 2>&1 | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('hint chunk64', d['hint_s_per_client'])"
