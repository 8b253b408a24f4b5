mkdir -p gpurun_out/r02k
O=gpurun_out/r02k
timeout 900 python -m pytest tests/test_gpu_seq.py tests/test_gpu_parity.py tests/test_gpu_edge.py -q -p no:cacheprovider -x > $O/pytest.log 2>&1
tail -2 $O/pytest.log





