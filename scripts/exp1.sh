mkdir -p gpurun_out
python scripts/exp_stack.py alexnet 0 '{}' '{"force_tile_planes":8}' '{"force_tile_planes":4,"force_stages":4}' >> gpurun_out/exp1.jsonl 2>&1
python scripts/exp_stack.py alexnet 1 '{}' '{"force_tile_planes":8}' >> gpurun_out/exp1.jsonl 2>&1
python scripts/exp_stack.py alexnet 2 '{}' '{"force_tile_planes":24}' '{"force_tile_planes":48}' '{"force_tile_planes":80}' >> gpurun_out/exp1.jsonl 2>&1
python scripts/exp_stack.py densenet121 120 '{}' '{"force_tile_planes":64}' '{"force_tile_planes":128}' '{"force_tile_planes":256}'  >> gpurun_out/exp1.jsonl 2>&1
timeout 900 python -m pytest tests -m gpu -q -x -k "tile_invariance or odd_shapes or random or golden or baseline" > gpurun_out/pytest_part.log 2>&1
