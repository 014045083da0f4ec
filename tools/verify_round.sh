set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 1200 python -m pytest tests -m gpu -x -q 2>&1 | tail -15 > gpurun_out/v_pytest.txt
timeout 300 python bench.py --steps 20 --warmup 3 > gpurun_out/v_bench.json 2> gpurun_out/v_bench.err
timeout 400 python tools/time_configs.py > gpurun_out/v_configs.txt 2>&1
