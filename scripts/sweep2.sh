#!/bin/bash
mkdir -p gpurun_out
for i in 0 1 2; do
  args=""
  for r in 2 4 7 14; do for p in 1 2 4 8 16; do for s in 4 8; do
    args="$args {\"force_rows_per_task\":$r,\"force_tile_planes\":$p,\"force_stages\":$s}"
  done; done; done
  timeout 600 python scripts/exp_stack.py alexnet $i '{}' $args
done > gpurun_out/sweep2.jsonl 2> gpurun_out/sweep2.err
