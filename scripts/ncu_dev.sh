#!/bin/bash
mkdir -p gpurun_out
NCU=/usr/local/cuda/bin/ncu
for spec in "alexnet 0" "resnet50 0" "vgg16 0" "densenet121 6"; do
  set -- $spec
  $NCU --set full --clock-control none --import-source on -k regex:'pool_cw|ew_kernel' -s 2 -c 1 \
     -o gpurun_out/prof_$1_$2 -f python scripts/prof_one.py $1 $2 4 > gpurun_out/ncu_$1_$2.log 2>&1
done
ls -la gpurun_out
