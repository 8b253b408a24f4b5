mkdir -p gpurun_out/r02q
O=gpurun_out/r02q
CS=/usr/local/cuda/bin/compute-sanitizer
timeout 900 python -m pytest tests/test_gpu_seq.py -q -p no:cacheprovider -x > $O/pytest.log 2>&1
tail -1 $O/pytest.log
timeout 600 $CS --tool racecheck --print-limit 20 python scripts/sanitize_families.py seq_fast seq_inplace seq_inplace_wide seq_halo seq_generic > $O/racecheck.log 2>&1
timeout 600 $CS --tool memcheck --leak-check full --print-limit 20 python scripts/sanitize_families.py ew staged seq_inplace > $O/memcheck.log 2>&1
grep -h "SUMMARY" $O/racecheck.log $O/memcheck.log
timeout 300 python scripts/exp_stack.py densenet121 120 '{}' copy > $O/final.jsonl 2>&1
timeout 300 python scripts/exp_sec51.py $O/sec51_56.jsonl 128 64 56 16 --no-eager > /dev/null 2>&1
