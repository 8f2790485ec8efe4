python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || exit 1
timeout 900 python -m pytest -q -x tests/test_gpu_protocol.py -m gpu 2>&1 | tail -15
