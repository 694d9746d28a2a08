mkdir -p gpurun_out
rm -f gpurun_out/small_ab.jsonl
for w in C1 C2 C1 C2; do
python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/small_ab.jsonl 2>> gpurun_out/small_ab.err
done
python bench.py --workload C4 --schedule single --steps 5 --warmup 3 --no-e2e --no-cpu-baseline >> gpurun_out/small_ab.jsonl 2>> gpurun_out/small_ab.err
python -m pytest tests -m gpu -x -q > gpurun_out/ab_tests.log 2>&1
tail -3 gpurun_out/ab_tests.log
