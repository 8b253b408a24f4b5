mkdir -p gpurun_out
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,memory.total --format=csv > gpurun_out/gpu.txt 2>&1
nproc >> gpurun_out/gpu.txt; lscpu | grep "Model name" >> gpurun_out/gpu.txt
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
timeout 1500 python -m pytest tests -m gpu -q -x --timeout 600 -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1
for wl in alexnet vgg16 resnet50 densenet121 c1; do
  timeout 600 python bench.py --workload $wl --out gpurun_out/bench_r1.jsonl > gpurun_out/bench_$wl.log 2>&1
done
tail -3 gpurun_out/pytest_gpu.log; cat gpurun_out/smoke.log | tail -3
