python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/build.log 2>&1; timeout 1200 python -m pytest tests -q -x -m gpu 2>&1 | tail -30
