timeout 300 python -m pytest tests/test_gpu_vm.py -q 2>&1 | tail -1
timeout 300 python scripts/vm_probe.py trace 2>&1 | grep "^ *[0-9]* \(gemm\|attn\|gn\|pool\|softmax\)" > gpurun_out/vm_ops.txt
cat gpurun_out/vm_ops.txt | python -c "
import sys,re,collections
agg=collections.defaultdict(lambda:[0,0.0])
for l in sys.stdin:
    m=re.match(r'\s*(\d+) (\w+)\s+items=\s*(\d+) S=\s*(\d+) wait=\s*([\d.]+) dur=\s*([\d.]+) end=\s*([\d.]+)\s*(.*)',l)
    if m: k=(m[2],m[8].strip()); agg[k][0]+=1; agg[k][1]+=float(m[6])+float(m[5])
print('total', sum(v[1] for v in agg.values()), 'ops', sum(v[0] for v in agg.values()))
for k,v in sorted(agg.items(), key=lambda x:-x[1][1])[:14]: print(f'{v[0]:3d}x {v[1]/v[0]:6.1f}us total {v[1]:6.1f}  {k[0]} {k[1]}')
"
