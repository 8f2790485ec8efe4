mkdir -p gpurun_out/final2
python -c "import __graft_entry__ as g; g.build(); g.smoke(); print('smoke ok')" > gpurun_out/final2/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 gpurun_out/final2/smoke.log
timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/final2/pytest.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/final2/pytest.log
timeout 600 python bench.py > gpurun_out/final2/bench.json 2> gpurun_out/final2/bench.err; echo "bench rc=$?"; cat gpurun_out/final2/bench.json
