#!/bin/bash
# Round-2 GPU check: smoke, GPU parity tests, compute-sanitizer over every kernel family,
# AlexNet per-stack timings (regression check of the staged item loop).
mkdir -p gpurun_out/r02a
O=gpurun_out/r02a
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $O/gpu.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck initcheck; do
  extra=""
  [ $tool = memcheck ] && extra="--leak-check full"
  timeout 900 $CS --tool $tool $extra --print-limit 50 python scripts/sanitize_families.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/sanitize_rc.txt
done
for i in 0 1 2; do
  timeout 300 python scripts/exp_stack.py alexnet $i '{}' copy
done > $O/alexnet_stacks.jsonl 2> $O/alexnet_stacks.err
tail -3 $O/pytest_gpu.log; tail -2 $O/smoke.log; cat $O/sanitize_rc.txt
