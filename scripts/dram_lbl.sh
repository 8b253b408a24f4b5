#!/bin/bash
# ncu DRAM bytes: fused stack vs torch eager layer by layer (all kernels after the inputs exist)
mkdir -p gpurun_out/lbl
for spec in "alexnet 0" "vgg16 0" "resnet50 0" "resnet50 1" "densenet121 13" "densenet121 120"; do
  set -- $spec
  /usr/local/cuda/bin/ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --cache-control all --clock-control none --csv --log-file gpurun_out/lbl/$1_$2.csv \
    python scripts/prof_lbl.py $1 $2 > gpurun_out/lbl/$1_$2.log 2>&1
done
