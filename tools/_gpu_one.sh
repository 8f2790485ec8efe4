# usage: bash tools/_gpu_one.sh <pytest args...>
python -c "from paper_2603_09190_b200 import build; build.build()" > gpurun_out/build.log 2>&1 || { tail -30 gpurun_out/build.log; exit 1; }
timeout 1200 python -m pytest -q -x "$@" 2>&1 | tail -40
