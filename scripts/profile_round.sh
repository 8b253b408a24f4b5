#!/bin/bash
# Collect the round's ncu evidence on the GPU box: launch list of the default bench, and one
# full capture of the dominant kernel of each workload (raw page exported to CSV on the box;
# only the AlexNet s1 report is kept, the rest stay under the 64 MiB return limit).
mkdir -p gpurun_out/prof
NCU=/usr/local/cuda/bin/ncu
$NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none \
     --csv --log-file gpurun_out/prof/launches_alexnet.csv \
     python bench.py --steps 3 --warmup 3 --no-cpu-baseline --no-lbl --no-graph --e2e-steps 1 > gpurun_out/prof/launches_alexnet.log 2>&1
for spec in "alexnet 0 staged" "alexnet 1 staged" "alexnet 2 staged" "vgg16 0 pool_vec" "resnet50 0 pool_vec" "densenet121 6 ew_kernel" "densenet121 13 pool_vec" "densenet121 120 staged"; do
  set -- $spec
  rep=/tmp/full_$1_$2
  $NCU --set full --clock-control none --import-source on -k regex:$3 -s 2 -c 1 \
     -o $rep -f python scripts/prof_one.py $1 $2 4 > gpurun_out/prof/full_$1_$2.log 2>&1
  $NCU -i $rep.ncu-rep --page raw --csv > gpurun_out/prof/full_$1_$2.raw.csv 2>/dev/null
  $NCU -i $rep.ncu-rep --page details --csv > gpurun_out/prof/full_$1_$2.details.csv 2>/dev/null
done
$NCU -i /tmp/full_alexnet_0.ncu-rep --page source --csv --print-source sass > gpurun_out/prof/full_alexnet_0.sass.csv 2>/dev/null
cp /tmp/full_alexnet_0.ncu-rep gpurun_out/prof/ 2>/dev/null
du -sh gpurun_out
