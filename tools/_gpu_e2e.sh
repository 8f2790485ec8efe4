#!/bin/bash
python -c "from paper_2603_09190_b200 import build; build.build()" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
python tools/e2e_split_sweep.py 8 0 4 8 12 16 2>&1 | tail -6
