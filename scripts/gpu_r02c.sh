#!/bin/bash
# Round-2: the new bench.py end to end (default run), and the 2-rank-on-1-GPU aggregation check.
mkdir -p gpurun_out/r02c
O=gpurun_out/r02c
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
BS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --no-extra --no-lbl --steps 50 > $O/bench_2rank_gloo.json 2> $O/bench_2rank_gloo.err
timeout 300 python bench.py --no-extra --no-lbl --steps 50 --no-cpu-baseline > $O/bench_1rank_short.json 2> $O/bench_1rank_short.err
tail -c 600 $O/bench_default.json; grep -E "Elapsed|Maximum resident" $O/bench_default.err
