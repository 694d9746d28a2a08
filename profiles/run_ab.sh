mkdir -p gpurun_out
rm -f gpurun_out/ab.jsonl
for i in 1 2 3; do
python bench.py --no-e2e --no-cpu-baseline >> gpurun_out/ab.jsonl 2>> gpurun_out/ab.err
done
