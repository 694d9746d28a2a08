mkdir -p gpurun_out
python -m pytest tests/test_ns.py tests/test_ns_multirank.py -m gpu -x -q > gpurun_out/ns_tests.log 2>&1
tail -2 gpurun_out/ns_tests.log
python profiles/ns_bench.py --configs C0,C1,C2,C3,C4 --steps 5 --warmup 2 2>&1 | python -c "
import sys,json
for l in sys.stdin:
    try: d=json.loads(l); print(d['config'], d['ms_per_iteration'])
    except Exception: print(l.strip()[:200])
"
