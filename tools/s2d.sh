out=gpurun_out/s2f; mkdir -p $out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -x -k tma > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 1200 python bench.py --tune-sizes 8192,1024,256 --tune-rounds 8 --config c2 > $out/ab_c2.jsonl 2>&1; echo "ab c2 rc=$?" >> $out/rc.txt
timeout 1200 python bench.py --tune-sizes 8192 --tune-rounds 8 --config c3 > $out/ab_c3.jsonl 2>&1; echo "ab c3 rc=$?" >> $out/rc.txt
