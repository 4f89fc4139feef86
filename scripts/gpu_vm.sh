timeout 300 python scripts/vm_probe.py trace > gpurun_out/vm_probe.txt 2>&1
timeout 300 python -m pytest tests/test_gpu_vm.py -q 2>&1 | grep -v "^E  *+" | tail -30 > gpurun_out/pytest_vm.txt
head -3 gpurun_out/vm_probe.txt; grep "time by" -A 100 gpurun_out/vm_probe.txt; cat gpurun_out/pytest_vm.txt
