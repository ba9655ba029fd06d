#!/bin/bash
# Developer A/B pass on one GPU box: build, bench lines of the named workloads
# (WL), optional env variants (AB="NAME=VAL ..."), then the GPU test suite.
# Usage: TAG=s2 WL="C2 C3" AB="FCFS_NEAREST_STAGED=1" bash tools/gpu_ab.sh
O=gpurun_out/${TAG:-ab}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
summ() { python -c "import json,sys;d=json.load(open('$1'));print('$1',round(d['ms_per_step']*1000,2),'us',round(d['roofline']['frac'],3),d['clocks']['sm_mhz'])" 2>&1 | tail -1; }
for w in ${WL:-C2 C3}; do
  for rep in 1 2; do
    timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/bench_${w}_$rep.json 2> $O/bench_${w}_$rep.err; summ $O/bench_${w}_$rep.json
    for v in $AB; do
      env $v timeout 300 python bench.py --workload $w --no-cpu-baseline --no-e2e > $O/bench_${w}_${v%%=*}_$rep.json 2> /dev/null; echo -n "$v: "; summ $O/bench_${w}_${v%%=*}_$rep.json
    done
  done
done
[ -n "$NO_TEST" ] || { timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -n 3 $O/pytest_gpu.log; }
