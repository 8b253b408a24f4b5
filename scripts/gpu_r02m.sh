mkdir -p gpurun_out/r02n
O=gpurun_out/r02n
timeout 900 python -m pytest tests/test_gpu_edge.py -q -p no:cacheprovider -x -k row_block > $O/pytest.log 2>&1
tail -2 $O/pytest.log
for i in 13 38 87 120; do timeout 300 python scripts/exp_stack.py densenet121 $i '{}' '{"force_generic":4}' '{"force_generic":4,"force_outputs_per_group":0}'; done > $O/rows.jsonl 2> $O/rows.err
for i in 0 1 2 3 4; do timeout 300 python scripts/exp_stack.py vgg16 $i '{}' '{"force_generic":4}'; done >> $O/rows.jsonl 2>> $O/rows.err
timeout 300 python scripts/exp_stack.py c1 0 '{}' '{"force_generic":4}' >> $O/rows.jsonl 2>> $O/rows.err
