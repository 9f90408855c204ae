timeout 900 python -m pytest tests/ -m gpu -x -q 2>&1 | tail -3
for i in 1 2; do
for L in _a ""; do
for P in bf16 fp16; do
MFG_GPU_LIB=libmfgpu$L.so timeout 300 python bench.py --steps 8 --warmup 3 --precision $P --no-cpu-baseline --no-other-precisions > /tmp/o.txt 2>/tmp/e.txt
python -c "import json,sys; d=json.loads(open('/tmp/o.txt').read().strip().splitlines()[-1]); r=d['roofline']['class_ms_share']; print('lib$L $P', round(d['value'],1), round(d['e2e']['value'],1), d['clocks']['sm_mhz'], round(d['ms_per_step'],2), {k: round(v*d['ms_per_step'],1) for k,v in r.items()}, d.get('parity'))" || tail -3 /tmp/e.txt
done; done; done
