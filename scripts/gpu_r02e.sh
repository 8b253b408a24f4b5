#!/bin/bash
mkdir -p gpurun_out/r02f
O=gpurun_out/r02f
timeout 900 python -m pytest tests/test_gpu_seq.py tests/test_gpu_parity.py -q -p no:cacheprovider -x -k "seq or sec51 or multi_sequence or random or graph or smem" > $O/pytest_seq.log 2>&1
tail -2 $O/pytest_seq.log
timeout 600 python scripts/exp_sec51.py $O/sec51_56.jsonl 128 64 56 1,16,40 --no-eager > /dev/null 2> $O/sec51_56.err
timeout 600 python scripts/exp_sec51.py $O/sec51_224.jsonl 32 64 224 8,16 --no-eager > /dev/null 2> $O/sec51_224.err
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:seq_staged -c 1 -o $O/seq16 -f python scripts/prof_sec51.py 16 0 2 > $O/ncu.log 2>&1
/usr/local/cuda/bin/ncu -i $O/seq16.ncu-rep --page details --csv > $O/seq16.details.csv 2>/dev/null
/usr/local/cuda/bin/ncu -i $O/seq16.ncu-rep --page source --csv --print-source sass > $O/seq16.sass.csv 2>/dev/null
ls -la $O
