mkdir -p gpurun_out
set -x
python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1
python -m pytest tests -m gpu -x -q > gpurun_out/gputests.log 2>&1; echo "pytest exit $?" >> gpurun_out/gputests.log
python bench.py > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err
python bench.py --impl reference --steps 3 --warmup 1 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
for w in C0 C1 C2 C3; do python bench.py --workload $w --steps 50 --warmup 5 --no-e2e --no-cpu-baseline >> gpurun_out/bench_small.jsonl 2>> gpurun_out/bench_small.err; done
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches_c4.csv python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_l.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:pair_tma -s 6 -c 2 -o gpurun_out/pair_c4 -f python bench.py --steps 2 --warmup 3 --no-e2e --no-cpu-baseline > gpurun_out/ncu_f.log 2>&1
tail -3 gpurun_out/gputests.log; cat gpurun_out/bench_c4.json
