mkdir -p gpurun_out
python -m pytest tests/test_ns.py tests/test_ns_multirank.py -m gpu -x -q > gpurun_out/ns_tests.log 2>&1
tail -2 gpurun_out/ns_tests.log
ncu --set full --clock-control none --import-source on -k regex:ns_stage -s 4 -c 2 -o gpurun_out/ns_c4 -f python profiles/ns_bench.py --configs C4 --steps 1 --warmup 1 > gpurun_out/ncu_ns4.log 2>&1
