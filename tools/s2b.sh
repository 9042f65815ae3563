out=gpurun_out/s2b; mkdir -p $out
timeout 900 python -m pytest tests/test_kernels_gpu.py -q -m gpu -k "tma or tuning" -x > $out/pytest_tma.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py --tune --tune-tma --steps 5 --config c2 > $out/tune_tma_c2.jsonl 2>&1; echo "tune c2 rc=$?" >> $out/rc.txt
timeout 900 python bench.py --tune --tune-tma --steps 5 --config c3 > $out/tune_tma_c3.jsonl 2>&1; echo "tune c3 rc=$?" >> $out/rc.txt
