mkdir -p gpurun_out
python scripts/exp_stack.py densenet121 13 copy '{}' '{"force_generic":3}' '{"force_generic":2}' >> gpurun_out/exp1.jsonl 2>&1
python scripts/exp_stack.py densenet121 87 '{}' '{"force_generic":3}' >> gpurun_out/exp1.jsonl 2>&1
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:pool_vec -s 2 -c 1 -o gpurun_out/prof_dn_t1 -f python scripts/prof_one.py densenet121 13 4 > /dev/null 2>&1
