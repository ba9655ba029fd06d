#!/bin/bash
# ncu --set full of one fused launch of each named config (tools/exp.py, 1 rep)
O=gpurun_out/${1:-ncu1}; shift
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; exit 1; }
for c in "$@"; do
  timeout 600 ncu --set full --clock-control none --import-source on -k regex:fcfs -s 3 -c 1 -o $O/full_$c -f \
    python tools/exp.py $c --reps 1 > $O/ncu_$c.log 2>&1; echo "ncu $c rc=$?"
done
