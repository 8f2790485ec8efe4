#!/bin/bash
python -c "from paper_2603_09190_b200 import build; build.build()" > /tmp/b.log 2>&1 || { tail /tmp/b.log; exit 1; }
timeout 600 python tools/batch_wire_profile.py 2>&1 | tail -45
