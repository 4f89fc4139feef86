timeout 300 python -m pytest tests/test_gpu_vm.py -q 2>&1 | tail -2
TRACE_OPS=3,29 timeout 300 python scripts/vm_probe.py trace > gpurun_out/vm_probe.txt 2>&1
head -1 gpurun_out/vm_probe.txt; grep "time by" -A 20 gpurun_out/vm_probe.txt | cut -c1-180
