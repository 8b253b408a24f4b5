mkdir -p gpurun_out/r02r
O=gpurun_out/r02r
for i in 13 38 87; do timeout 300 python scripts/exp_stack.py densenet121 $i '{}' '{"force_generic":3}' '{"force_generic":3,"force_stages":3}' '{"force_generic":3,"force_stages":2}'; done > $O/t.jsonl 2>&1
