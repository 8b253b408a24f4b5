mkdir -p gpurun_out/r02h
O=gpurun_out/r02h
timeout 900 python -m pytest tests/test_gpu_seq.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -p no:cacheprovider -x > $O/pytest.log 2>&1
tail -2 $O/pytest.log
timeout 600 python scripts/exp_sec51.py $O/sec51_56.jsonl 128 64 56 1,16,40 > /dev/null 2> $O/e1.err
BS_SEC51_OPTS='{"force_stages": 2}' timeout 600 python scripts/exp_sec51.py $O/sec51_56_s2.jsonl 128 64 56 16 --no-eager > /dev/null 2> $O/e2.err
timeout 600 python scripts/exp_sec51.py $O/sec51_112.jsonl 64 64 112 16,40 --no-eager > /dev/null 2> $O/e3.err
timeout 600 python scripts/exp_sec51.py $O/sec51_28.jsonl 256 64 28 16 --no-eager > /dev/null 2> $O/e4.err
/usr/local/cuda/bin/ncu --set full --clock-control none --import-source on -k regex:seq_ -c 1 -o $O/seq16 -f python scripts/prof_sec51.py 16 0 2 > $O/ncu.log 2>&1
/usr/local/cuda/bin/ncu -i $O/seq16.ncu-rep --page details --csv > $O/seq16.details.csv 2>/dev/null
/usr/local/cuda/bin/ncu -i $O/seq16.ncu-rep --page source --csv --print-source sass > $O/seq16.sass.csv 2>/dev/null
