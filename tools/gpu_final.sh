#!/bin/bash
# Final check on one box: build, the GPU test suite, smoke, the default bench line.
O=gpurun_out/${TAG:-final}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -q > $O/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -n 3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -n 2 $O/smoke.log
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench rc=$?"
python -c "import json;d=json.load(open('$O/bench_default.json'));print(d['config']['workload'],d['ms_per_step'],d['roofline']['frac'],d['e2e']['value'],d['clocks'])"
