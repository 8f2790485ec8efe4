#!/bin/bash
ZPIR_NVCC_EXTRA=-DZPIR_TC_TRACE python -c "from paper_2603_09190_b200 import build; build.build(force=True)" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
python tools/tc_trace.py 2>&1 | tail -45
