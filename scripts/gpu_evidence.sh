#!/bin/bash
# Round evidence on one B200: tests, sanitizers, bench (default + 2-rank gloo), §5.1 sweeps,
# ncu launch list / DRAM traffic / full captures.  Output: gpurun_out/$TAG/
TAG=${TAG:-r02_final}
O=gpurun_out/$TAG
mkdir -p $O
NCU=/usr/local/cuda/bin/ncu
CS=/usr/local/cuda/bin/compute-sanitizer
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total,driver_version --format=csv > $O/gpu.txt 2>&1
nproc > $O/nproc.txt; lscpu | grep -E "Model name|^CPU\(s\)" >> $O/nproc.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > $O/pytest_gpu.log 2>&1
tail -1 $O/pytest_gpu.log
if [ -z "$NOSAN" ]; then
for tool in memcheck racecheck synccheck initcheck; do
  extra=""; [ $tool = memcheck ] && extra="--leak-check full"
  timeout 1200 $CS --tool $tool $extra --print-limit 50 python scripts/sanitize_families.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/sanitize_rc.txt
done
fi
if [ -z "$NOBENCH" ]; then
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err
BS_BENCH_BACKEND=gloo timeout 600 python -m torch.distributed.run --nnodes=1 --nproc-per-node 2 --master-addr 127.0.0.1 --master-port 29533 bench.py --gpus 2 --no-extra --no-lbl --steps 50 > $O/bench_2rank_gloo.json 2> $O/bench_2rank_gloo.err
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > $O/bench_reference.json 2> $O/bench_reference.err
fi
if [ -z "$NOSEC" ]; then
timeout 900 python scripts/exp_sec51.py $O/sec51_56.jsonl 128 64 56 1,2,4,8,12,16,17,20,24,32,40 > /dev/null 2> $O/sec51_56.err
timeout 900 python scripts/exp_sec51.py $O/sec51_64.jsonl 128 64 64 1,16,40 --no-eager > /dev/null 2> $O/sec51_64.err
timeout 900 python scripts/exp_sec51.py $O/sec51_112.jsonl 64 64 112 1,5,16,32,40 --no-eager > /dev/null 2> $O/sec51_112.err
timeout 900 python scripts/exp_sec51.py $O/sec51_224.jsonl 32 64 224 1,5,8,15,16,30,40 --no-eager > /dev/null 2> $O/sec51_224.err
# the paper's cache-limit artifact: 224^2 planes under a 110 KB budget -> halo tiles
BS_SEC51_OPTS='{"smem_budget_bytes": 112640}' timeout 900 python scripts/exp_sec51.py $O/sec51_224_budget110k.jsonl 32 64 224 1,5,8,14,15,16,30,40 --no-eager > /dev/null 2> $O/sec51_224_budget.err
fi
if [ -z "$NONCU" ]; then
# launch list of a short default bench (cold-cache, serialised: compare shares)
[ -z "$NOFULL" ] && $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
     --log-file $O/launches_resnet50.csv python bench.py --steps 2 --warmup 3 --no-extra --no-lbl --no-per-stack \
     --no-cpu-baseline --no-validate --e2e-steps 1 > $O/launches_resnet50.log 2>&1
# DRAM traffic per launch of each workload's dominant stack (cold cache)
for spec in "resnet50 0" "alexnet 0" "vgg16 0" "densenet121 11"; do
  set -- $spec
  $NCU --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv \
       --log-file $O/traffic_$1_$2.csv python scripts/prof_one.py $1 $2 3 > $O/traffic_$1_$2.log 2>&1
done
[ -n "$NOFULL" ] && { du -sh $O; exit 0; }   # (NOFULL=1: the traffic captures only)
for spec in "resnet50 0 pool_vec" "alexnet 0 pool_staged" "densenet121 11 ew_kernel" "densenet121 -1 pool_planes"; do
  set -- $spec
  $NCU --set full --clock-control none --import-source on -k regex:$3 -s 1 -c 1 -o /tmp/full_$1_$2 -f \
       python scripts/prof_one.py $1 $2 3 > $O/full_$1_$2.log 2>&1
  $NCU -i /tmp/full_$1_$2.ncu-rep --page details --csv > $O/full_$1_$2.details.csv 2>/dev/null
  $NCU -i /tmp/full_$1_$2.ncu-rep --page raw --csv > $O/full_$1_$2.raw.csv 2>/dev/null
done
$NCU --set full --clock-control none --import-source on -k regex:seq_ -c 1 -o /tmp/full_seq16 -f \
     python scripts/prof_sec51.py 16 0 2 > $O/full_seq16.log 2>&1
$NCU -i /tmp/full_seq16.ncu-rep --page details --csv > $O/full_seq16.details.csv 2>/dev/null
$NCU -i /tmp/full_seq16.ncu-rep --page raw --csv > $O/full_seq16.raw.csv 2>/dev/null
fi
du -sh $O
