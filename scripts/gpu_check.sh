#!/bin/bash
# GPU round-trip used during development: smoke, GPU parity tests, bench lines.
mkdir -p gpurun_out
WL=${WL:-"alexnet vgg16 resnet50 densenet121 c1"}
TAG=${TAG:-dev}
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
if [ -z "$NOTEST" ]; then
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
fi
for wl in $WL; do
  timeout 600 python bench.py --workload $wl $BENCHARGS --out gpurun_out/bench_$TAG.jsonl > gpurun_out/bench_$wl.log 2>&1
done
tail -3 gpurun_out/pytest_gpu.log; tail -2 gpurun_out/smoke.log
