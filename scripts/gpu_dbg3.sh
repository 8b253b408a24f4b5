export BS_VALIDATE_ALL=1
python bench.py --no-lbl --no-per-stack --no-cpu-baseline --steps 50 > gpurun_out/dbg3.json 2>gpurun_out/dbg3.err
python -c "
import json
d=json.loads(open('gpurun_out/dbg3.json').read())
print('resnet50', d['validation']['ok'], d['roofline']['frac'], d['roofline']['avg_launch_ms'])
for wl,w in d['workloads'].items():
    if wl!='c1': print(wl, w['validation']['ok'], len(w['validation']['errors']), w['roofline']['frac'], [e[:50] for e in w['validation']['errors']][:5])
"
