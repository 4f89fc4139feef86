set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm --format=csv
python -m pytest tests -m gpu -x -q 2>&1 | tail -30 > gpurun_out/pytest_gpu.txt
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.txt 2>&1
timeout 600 python bench.py --precision bf16 --steps 20 --warmup 3 --no-cpu > gpurun_out/bench_bf16.json 2> gpurun_out/bench_bf16.err
cat gpurun_out/pytest_gpu.txt gpurun_out/smoke.txt gpurun_out/bench_bf16.json; tail -5 gpurun_out/bench_bf16.err
