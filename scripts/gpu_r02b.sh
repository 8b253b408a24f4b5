#!/bin/bash
# Round-2: racecheck + timing of the empty-barrier protocol variants (see k_pool_staged.cu).
mkdir -p gpurun_out/r02b
O=gpurun_out/r02b
CS=/usr/local/cuda/bin/compute-sanitizer
for v in default arrive_all proxy_fence; do
  if [ "$v" = "default" ]; then unset BS_LIB; else export BS_LIB=$PWD/paper_1804_08378_b200/libbrainslug_$v.so; fi
  timeout 600 $CS --tool racecheck --print-limit 20 python scripts/sanitize_families.py staged staged_avg7 seq_fast seq_generic > $O/racecheck_$v.log 2>&1
  for i in 0 1 2; do
    timeout 300 python scripts/exp_stack.py alexnet $i '{}' | sed "s/^{/{\"variant\": \"$v\", /"
  done >> $O/alexnet_variants.jsonl 2>> $O/alexnet_variants.err
done
unset BS_LIB
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider -x > $O/pytest_gpu.log 2>&1
for tool in memcheck synccheck initcheck; do
  timeout 900 $CS --tool $tool --print-limit 50 python scripts/sanitize_families.py > $O/sanitize_$tool.log 2>&1
  echo "$tool rc=$?" >> $O/sanitize_rc.txt
done
tail -3 $O/pytest_gpu.log; cat $O/sanitize_rc.txt; grep -c "Race reported" $O/racecheck_*.log
