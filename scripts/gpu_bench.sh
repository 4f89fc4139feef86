nproc; lscpu | grep "Model name"
timeout 900 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; cat gpurun_out/bench_default.json; tail -3 gpurun_out/bench_default.err
timeout 600 python bench.py --sweep --no-cpu --steps 20 > gpurun_out/bench_sweep.json 2>/dev/null; python -c "import json; d=json.load(open('gpurun_out/bench_sweep.json')); print(json.dumps(d['sweep']))"
timeout 900 python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2>&1; tail -1 gpurun_out/bench_ref.json
