mkdir -p gpurun_out
timeout 600 python scripts/exp_stack.py alexnet 0 '{}' '{"force_rows_per_task":14}' '{"force_rows_per_task":7}' '{"force_rows_per_task":4}' '{"force_tile_planes":1,"force_stages":8,"force_rows_per_task":7}' '{"force_tile_planes":1,"force_stages":8,"force_rows_per_task":4}' '{"force_tile_planes":2,"force_stages":4,"force_rows_per_task":7}' >> gpurun_out/exp1.jsonl 2>&1
timeout 600 python scripts/exp_stack.py alexnet 1 '{}' '{"force_rows_per_task":7}' '{"force_rows_per_task":4}' '{"force_tile_planes":4,"force_rows_per_task":4}' >> gpurun_out/exp1.jsonl 2>&1
timeout 600 python scripts/exp_stack.py alexnet 2 '{}' '{"force_rows_per_task":3}' '{"force_rows_per_task":2}' >> gpurun_out/exp1.jsonl 2>&1
