#!/bin/bash
# Dev: default bench line (per workload in $WLS) for each library variant in $VARIANTS.
mkdir -p gpurun_out
for v in $VARIANTS; do
  if [ "$v" = "default" ]; then unset BS_LIB; else export BS_LIB=$PWD/paper_1804_08378_b200/libbrainslug_$v.so; fi
  for wl in ${WLS:-alexnet}; do
    timeout 600 python bench.py --workload $wl --no-lbl --no-cpu-baseline $BENCHARGS | sed "s/^{/{\"variant\": \"$v\", /"
  done
done > gpurun_out/bench_variants.jsonl 2> gpurun_out/bench_variants.err
