#!/bin/bash
python -c "from paper_2603_09190_b200 import build; build.build()" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
PYTHONPATH=. timeout 600 python tools/wire_breakdown.py 2>&1 | tail -25
