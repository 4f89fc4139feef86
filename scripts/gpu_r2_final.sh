# Round-2 evidence: bench line, reference arm, launch lists, ncu captures (summaries under gpurun_out/)
set -x
mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,clocks_event_reasons.active --format=csv
timeout 1200 python bench.py --steps 20 --warmup 5 > gpurun_out/bench_r02.json 2> gpurun_out/bench_r02.err
timeout 600 python scripts/step_table.py --R 64 --out gpurun_out/step_table_r02.txt > /dev/null 2>&1
# ncu launch list of one graph-replayed batch-1 step (cold-cache, serialised: compare shares)
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --profile-from-start off --csv \
    --log-file gpurun_out/launches_step1_r02.csv python scripts/prof_step.py > /dev/null 2>&1
# --set full of the batch-1 L0 gated conv (DRAM traffic of the roofline line) and of the halo conv at R=64
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_tc_kernel -s 1 -c 1 \
    -o /tmp/gated_conv python scripts/prof_step.py > /dev/null 2>&1
ncu -i /tmp/gated_conv.ncu-rep --page raw --csv > gpurun_out/ncu_gated_conv_raw.csv 2>/dev/null
timeout 900 ncu --set full --import-source on --clock-control none --profile-from-start off -k regex:gemm_halo -s 0 -c 2 \
    -o /tmp/halo_conv python scripts/prof_step_batched.py 64 > /dev/null 2>&1
ncu -i /tmp/halo_conv.ncu-rep --page raw --csv > gpurun_out/ncu_halo_conv_raw.csv 2>/dev/null
ncu -i /tmp/halo_conv.ncu-rep --page details --csv > gpurun_out/ncu_halo_conv_details.csv 2>/dev/null
# HBM-class kernels of the batch-1 step: DRAM bytes + duration
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_bytes.sum --clock-control none \
    --profile-from-start off -k regex:"gn_|pool2|mask|softmax|materialize" --csv --log-file gpurun_out/ncu_hbm_kernels.csv \
    python scripts/prof_step.py > /dev/null 2>&1
ls -la gpurun_out; tail -3 gpurun_out/bench_r02.err
