out=gpurun_out/s2c; mkdir -p $out
timeout 900 python -m pytest tests/test_kernels_gpu.py tests/test_stream_gpu.py -q -m gpu -x > $out/pytest.log 2>&1; echo "pytest rc=$?" >> $out/rc.txt
timeout 900 python bench.py --tune-sizes --config c2 > $out/tune_sizes_c2.jsonl 2>&1; echo "tune sizes rc=$?" >> $out/rc.txt
timeout 600 python bench.py --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $out/bench.json 2> $out/bench.err; echo "bench rc=$?" >> $out/rc.txt
timeout 600 python bench.py --config c3 --steps 20 --warmup 5 --no-e2e --no-cpu-baseline > $out/bench_c3.json 2>> $out/bench.err; echo "bench c3 rc=$?" >> $out/rc.txt
