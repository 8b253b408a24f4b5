#!/bin/bash
# Round-2: new sequence kernel (vectorised fast path + halo tiles): GPU tests, §5.1 timings.
mkdir -p gpurun_out/r02d
O=gpurun_out/r02d
timeout 900 python -m pytest tests/test_gpu_seq.py -q -p no:cacheprovider -x > $O/pytest_seq.log 2>&1
tail -3 $O/pytest_seq.log
timeout 600 python scripts/exp_sec51.py $O/sec51_56.jsonl 128 64 56 1,4,8,16,17,40 > /dev/null 2> $O/sec51_56.err
timeout 600 python scripts/exp_sec51.py $O/sec51_224.jsonl 32 64 224 1,5,15,16,30,40 --no-eager > /dev/null 2> $O/sec51_224.err
timeout 600 python scripts/exp_sec51.py $O/sec51_112.jsonl 64 64 112 1,5,16,40 --no-eager > /dev/null 2> $O/sec51_112.err
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
tail -3 $O/pytest_gpu.log
