mkdir -p gpurun_out
python profiles/ns_bench.py --configs C0,C1,C2,C3,C4 --steps 5 --warmup 2 --out gpurun_out/ns_bench.json > gpurun_out/ns_bench.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ns_stage -s 4 -c 1 -o gpurun_out/ns_c4 -f python profiles/ns_bench.py --configs C4 --steps 1 --warmup 1 > gpurun_out/ncu_ns4.log 2>&1
ncu --set full --clock-control none --import-source on -k regex:ns_stage -s 4 -c 1 -o gpurun_out/ns_c3 -f python profiles/ns_bench.py --configs C3 --steps 1 --warmup 1 > gpurun_out/ncu_ns3.log 2>&1
cat gpurun_out/ns_bench.log
