mkdir -p gpurun_out/r02g
O=gpurun_out/r02g
for P in 1 2 4; do
  BS_SEC51_OPTS="{\"force_tile_planes\": $P}" timeout 600 python scripts/exp_sec51.py - 128 64 56 16 --no-eager | sed "s/^{/{\"P\": $P, /" >> $O/sweep.jsonl
done
