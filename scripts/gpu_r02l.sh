mkdir -p gpurun_out/r02l
O=gpurun_out/r02l
for i in 13 38 87; do
  timeout 300 python scripts/exp_stack.py densenet121 $i '{}' '{"force_generic":3}' '{"force_generic":2}' '{"force_generic":3,"force_stages":4}' '{"force_generic":1}'
done > $O/trans.jsonl 2> $O/trans.err
timeout 300 python scripts/exp_stack.py densenet121 120 '{}' '{"force_stages":2}' '{"force_stages":4}' '{"force_tile_planes":32}' '{"force_tile_planes":128}' '{"force_tile_planes":256}' '{"force_generic":2}' '{"force_generic":1}' > $O/final.jsonl 2> $O/final.err
timeout 300 python scripts/exp_stack.py vgg16 4 '{}' '{"force_generic":3}' '{"force_generic":2}' >> $O/final.jsonl 2>> $O/final.err
timeout 300 python scripts/exp_stack.py alexnet 2 '{}' '{"force_stages":3}' '{"force_tile_planes":10}' '{"force_tile_planes":40}' >> $O/final.jsonl 2>> $O/final.err
