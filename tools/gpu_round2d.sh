#!/bin/bash
mkdir -p gpurun_out
timeout 900 python -m pytest tests/test_gpu_coarse_bf16.py tests/test_gpu_gates.py tests/test_gpu_vsa_full.py -q -x -p no:cacheprovider > gpurun_out/pytest_d.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_d.log
timeout 300 python bench.py --no-cpu > gpurun_out/bench_d.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_d.log
timeout 300 python bench.py --no-cpu --coarse bf16 > gpurun_out/bench_d2.log 2>&1; echo "bench rc=$?" >> gpurun_out/bench_d2.log
tail -30 gpurun_out/pytest_d.log
for f in bench_d bench_d2; do python -c "
import json; d=[json.loads(l) for l in open('gpurun_out/$f.log') if l.startswith('{')][0]
print(d['coarse_mode'], d['ms_per_step'], d['value'], {k: v['ms'] for k, v in d['stages'].items()}, d['other_coarse_mode'])"; done
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_bf16coarse.csv python -c "
import sys; sys.path.insert(0,'.')
import torch, paper_2505_13389_b200 as vsa
L = vsa.TileLayout(21, 30, 52, pad=True)
op = vsa.VsaOp(L, 1, 12, 128, 78, coarse='bf16')
x = [torch.randn((1, 12, L.seq_len, 128), device='cuda').bfloat16() for _ in range(6)]
for _ in range(2):
    op.forward(*x[:5]); op.backward(x[5])
torch.cuda.synchronize()
" > /dev/null 2>&1
python - <<'PY'
import csv
rows = list(csv.reader(open('gpurun_out/launches_bf16coarse.csv')))
hdr = None
for r in rows:
    if 'Kernel Name' in r: hdr = r; continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum': print(d['Kernel Name'][:50], d['Metric Value'])
PY
