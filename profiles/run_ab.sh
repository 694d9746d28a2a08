mkdir -p gpurun_out
rm -f gpurun_out/small_ab.jsonl
for w in C1 C1 C2; do
python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/small_ab.jsonl 2>> gpurun_out/small_ab.err
done
python bench.py --workload C1 --tile-rows 16 --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/small_ab.jsonl 2>> gpurun_out/small_ab.err
python bench.py --workload C0 --schedule single --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/small_ab.jsonl 2>> gpurun_out/small_ab.err
python -m pytest tests/test_gpu_parity.py tests/test_gpu_kernels.py tests/test_gpu_fulllength.py -m gpu -x -q > gpurun_out/ab_tests.log 2>&1
tail -3 gpurun_out/ab_tests.log
