#!/bin/bash
# Dev: AlexNet per-stack timings for each library variant named in $VARIANTS ("" = default lib).
mkdir -p gpurun_out
for v in $VARIANTS; do
  if [ "$v" = "default" ]; then unset BS_LIB; else export BS_LIB=$PWD/paper_1804_08378_b200/libbrainslug_$v.so; fi
  for i in 0 1 2; do
    timeout 300 python scripts/exp_stack.py alexnet $i '{}' ${EXTRA_OPTS} | sed "s/^{/{\"variant\": \"$v\", /"
  done
done > gpurun_out/variants.jsonl 2> gpurun_out/variants.err
