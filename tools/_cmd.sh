timeout 600 python -m pytest tests -m gpu -x -q 2>&1 | tail -2
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/b.json 2>gpurun_out/b.err; echo "bench $?"
python -c "
import json; d=json.load(open('gpurun_out/b.json')); c=d['config5']
print(d['value'], d['e2e']['value'], d['batched']['value'])
for k in ('householder_pair','sparse_sign'): print(k, c[k]['ms_per_call'], c[k]['multiplier_apply'])
"
