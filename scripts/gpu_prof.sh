timeout 600 ncu --set full --import-source on --profile-from-start off --kernel-name regex:gemm_tc_kernel --launch-count 1 -o gpurun_out/gated_conv python scripts/prof_conv.py > gpurun_out/ncu_conv.log 2>&1
tail -2 gpurun_out/ncu_conv.log
