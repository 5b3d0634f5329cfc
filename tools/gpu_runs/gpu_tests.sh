# usage: bash tools/gpu_runs/gpu_tests.sh <pytest args...>
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv,noheader
timeout 1500 python -m pytest "$@" 2>&1 | tail -60
