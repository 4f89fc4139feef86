# Round-2 final evidence (after the short-run attention / TMA attention epilogue / GN work):
# bench line, step tables, batch-1 launch list, ncu of the short-run attention in the stacked step
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_final.json 2> gpurun_out/bench_final.err
timeout 600 python scripts/step_table.py --R 64 --out gpurun_out/step_tables_final.txt > /dev/null 2>&1
timeout 600 ncu -f --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_step1_final.csv python scripts/prof_step.py > /dev/null 2>&1
# short-run attention kernels of one stacked step: duration, DRAM / L2 bytes, L2 hit rate, issue activity
timeout 900 ncu -f --clock-control none --cache-control none --profile-from-start off -k regex:attn_short --csv \
    --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum,lts__t_sector_hit_rate.pct,sm__cycles_active.avg,sm__throughput.avg.pct_of_peak_sustained_elapsed \
    --log-file gpurun_out/ncu_attn_short_R64.csv python scripts/prof_step_batched.py > /dev/null 2>&1
ls -la gpurun_out; tail -3 gpurun_out/bench_final.err
