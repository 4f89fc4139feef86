# Round-2 final evidence: bench line, reference arm, step tables, launch list, ncu of the gated conv
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 900 python bench.py --impl reference --steps 4 --warmup 1 > gpurun_out/bench_reference_final.json 2> gpurun_out/bench_reference_final.err
timeout 600 python scripts/step_table.py --R 64 --out gpurun_out/step_tables_final.txt > /dev/null 2>&1
timeout 600 ncu -f --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_step1_final.csv python scripts/prof_step.py > /dev/null 2>&1
timeout 900 ncu -f --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_tc_kernel -s 1 -c 1 \
    -o /tmp/gated_conv python scripts/prof_step.py > /dev/null 2>&1
ncu -i /tmp/gated_conv.ncu-rep --page raw --csv > gpurun_out/ncu_gated_conv_raw_final.csv 2>/dev/null
ls -la gpurun_out; tail -3 gpurun_out/bench_final.err
