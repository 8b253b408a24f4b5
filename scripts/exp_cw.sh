mkdir -p gpurun_out
for v in "" _cw12 _cw16; do
  if [ -n "$v" ]; then export BS_LIB=$PWD/paper_1804_08378_b200/libbrainslug$v.so; else unset BS_LIB; fi
  timeout 600 python bench.py --workload alexnet --no-cpu-baseline --per-stack --no-lbl --out gpurun_out/exp_cw$v.jsonl > /dev/null 2>&1
done
