#!/bin/bash
# Parameter sweep of the staged pool kernel on the AlexNet stacks (dev experiment).
mkdir -p gpurun_out
nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/tma_ceiling scripts/tma_ceiling.cu
for b in 99123200 71663616 22151168; do echo "bytes $b"; /tmp/tma_ceiling $b; done > gpurun_out/tma_ceiling.txt 2>&1
for i in 0 1 2; do
  timeout 300 python scripts/exp_stack.py alexnet $i copy '{}' \
    '{"force_tile_planes":1}' '{"force_tile_planes":2}' '{"force_tile_planes":4}' '{"force_tile_planes":8}' \
    '{"force_tile_planes":1,"force_stages":8}' '{"force_tile_planes":2,"force_stages":6}' \
    '{"force_stages":2}' '{"force_stages":4}' '{"force_generic":2}' '{"force_generic":1}'
done > gpurun_out/sweep_alexnet.jsonl 2> gpurun_out/sweep_alexnet.err
