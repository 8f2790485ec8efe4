#!/bin/bash
python -c "from paper_2603_09190_b200 import build; build.build()" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
for i in 1 2; do
python tools/split_sweep.py 36 30 34 36 38 2>&1 | tail -4
done
timeout 600 python -m pytest tests/test_gpu_kernels.py tests/test_gpu_parity.py tests/test_gpu_protocol.py tests/test_gpu_db_api.py -q -m gpu -x 2>&1 | tail -3
