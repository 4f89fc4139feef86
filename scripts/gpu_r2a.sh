set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
timeout 900 python -m pytest tests/test_gpu_c2_parity.py -x -q -s 2>&1 | tail -40 > gpurun_out/pytest_c2.txt
timeout 900 python -m pytest tests -m gpu -q 2>&1 | tail -15 > gpurun_out/pytest_gpu.txt
timeout 900 python bench.py --steps 20 --warmup 5 > gpurun_out/bench.json 2> gpurun_out/bench.err
cat gpurun_out/pytest_c2.txt gpurun_out/pytest_gpu.txt; tail -c 3000 gpurun_out/bench.json; tail -20 gpurun_out/bench.err
