#!/bin/bash
# Quick GPU iteration: parity tests + kernel timings (tools/exp.py).
O=gpurun_out/${1:-quick}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; tail -30 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q 2>&1 | tail -15; echo "pytest gpu rc=${PIPESTATUS[0]}"
timeout 600 python tools/exp.py ${EXP_CFGS:-C3 C4a C4b C5 C2a C2b} --reps 30 ${EXP_ARGS}
