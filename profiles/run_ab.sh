mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
for i in 1 2; do
python bench.py --no-e2e --no-cpu-baseline >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
python bench.py --workload C3 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
python -m pytest tests/test_gpu_parity.py tests/test_gpu_fullsize.py tests/test_gpu_fulllength.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1
tail -3 gpurun_out/ab_tests.log
