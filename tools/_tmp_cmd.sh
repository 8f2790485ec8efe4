for c in 0 40; do
  ZPIR_COMPRESS_CTAS=$c python bench.py --no-cpu-baseline --no-extra-e2e --e2e-steps 5 2>gpurun_out/err_$c.txt | tail -1 | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('ctas=$c bench', round(d['value']), round(d['ms_per_step']*1e3,1), round(d['roofline'].get('ms_in_step',0)*1e3,1), d['clocks']['sm_mhz'])"
done
tail -3 gpurun_out/err_0.txt
