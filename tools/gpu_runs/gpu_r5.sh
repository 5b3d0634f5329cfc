nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_radau5.py -x -q 2>&1 | tail -30
timeout 600 python bench.py --config 2 --steps 3 --warmup 3 2>&1 | tail -5
