timeout 300 python -m pytest tests -m gpu -q -x 2>&1 | tail -1
for R in 4 8 16; do timeout 600 python bench.py --no-cpu --steps 20 --requests $R 2>/dev/null | python -c "import json,sys; d=json.loads(sys.stdin.read()); print('R=$R', d['ms_per_step'], d['batched'])"; done
