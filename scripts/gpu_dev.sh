#!/bin/bash
# Dev round-trip: GPU tests, AlexNet per-stack timings under a few plan options, default bench.
mkdir -p gpurun_out
timeout 900 python -m pytest tests -m gpu -q -x -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
for i in 0 1 2; do
  timeout 300 python scripts/exp_stack.py alexnet $i '{}' ${EXTRA_OPTS}
done > gpurun_out/dev_alexnet.jsonl 2> gpurun_out/dev_alexnet.err
timeout 600 python bench.py --no-lbl > gpurun_out/bench_dev_default.json 2> gpurun_out/bench_dev_default.err
tail -3 gpurun_out/pytest_gpu.log
