#!/bin/bash
mkdir -p gpurun_out
for v in $VARIANTS; do
  if [ "$v" = "default" ]; then unset BS_LIB; else export BS_LIB=$PWD/paper_1804_08378_b200/libbrainslug_$v.so; fi
  for d in 8 16; do python scripts/exp_seq_opts.py $d "{}" | sed "s/^{/{\"variant\": \"$v\", /"; done
done > gpurun_out/seq_variants.jsonl 2>&1
