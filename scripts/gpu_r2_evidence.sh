# Round-2 (second half) evidence: bench line, step tables, ncu of the CTA-pair conv and the halo conv
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02b.json 2> gpurun_out/bench_r02b.err
timeout 600 python scripts/step_table.py --R 64 --out gpurun_out/step_tables_r02b.txt > /dev/null 2>&1
# ncu launch list of one graph-replayed batch-1 step
timeout 600 ncu -f --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_step1_r02b.csv python scripts/prof_step.py > /dev/null 2>&1
# tensor-pipe / DRAM metrics of every persistent GEMM launch of the 64-request step: CTA-pair
# kernel (default) and the single-SM kernel for the same GEMMs (FIS_PAIR=0)
M=gpu__time_duration.sum,sm__pipe_tensor_subpipe_hmma_cycles_active.avg.pct_of_peak_sustained_active,dram__bytes_read.sum,dram__bytes_write.sum
timeout 900 ncu -f --metrics $M --clock-control none --profile-from-start off -k regex:"gemm_pair|gemm_big|gemm_halo" --csv \
    --log-file gpurun_out/ncu_gemms_R64_pair.csv python scripts/prof_step_batched.py 64 > /dev/null 2>&1
FIS_PAIR=0 timeout 900 ncu -f --metrics $M --clock-control none --profile-from-start off -k regex:"gemm_pair|gemm_big|gemm_halo" --csv \
    --log-file gpurun_out/ncu_gemms_R64_single.csv python scripts/prof_step_batched.py 64 > /dev/null 2>&1
# --set full of the batch-1 L0 gated conv (roofline traffic)
timeout 900 ncu -f --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_tc_kernel -s 1 -c 1 \
    -o /tmp/gated_conv python scripts/prof_step.py > /dev/null 2>&1
ncu -i /tmp/gated_conv.ncu-rep --page raw --csv > gpurun_out/ncu_gated_conv_raw_b.csv 2>/dev/null
ls -la gpurun_out; tail -3 gpurun_out/bench_r02b.err
