#!/bin/bash
# Sequence-kernel iteration: GPU sequence tests + §5.1 timings at 56^2 / 112^2 (+ 224^2 with FULL=1).
O=gpurun_out/${TAG:-seq}
mkdir -p $O
timeout 900 python -m pytest tests/test_gpu_seq.py -q -x -p no:cacheprovider > $O/pytest_seq.log 2>&1; tail -2 $O/pytest_seq.log
timeout 600 python scripts/exp_sec51.py $O/sec51_56.jsonl 128 64 56 1,16,40 --no-eager > /dev/null 2> $O/sec51_56.err
timeout 600 python scripts/exp_sec51.py $O/sec51_112.jsonl 64 64 112 16,40 --no-eager > /dev/null 2> $O/sec51_112.err
[ -n "$FULL" ] && timeout 900 python scripts/exp_sec51.py $O/sec51_224.jsonl 32 64 224 5,16,40 --no-eager > /dev/null 2> $O/sec51_224.err
python - <<PY
import json
for f in ("56","112","224"):
    try:
        for l in open("$O/sec51_%s.jsonl"%f): 
            d=json.loads(l); print(f, d["depth"], {k:round(v["us_per_block"],2) for k,v in d.items() if isinstance(v,dict) and "us_per_block" in v})
    except FileNotFoundError: pass
PY
