#!/bin/bash
# Developer ncu pass: --set full of one workload's fcfs kernels, summarised on the box.
# Usage: TAG=s4 W=C2 bash tools/gpu_ncu.sh
O=gpurun_out/${TAG:-ncu}
mkdir -p $O
W=${W:-C2}
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fcfs -s 4 -c 1 -o $O/full_$W -f \
  python bench.py --workload $W --steps 2 --warmup 3 --soak-s 0 --no-e2e --no-cpu-baseline > $O/ncu_full_$W.log 2>&1; echo "ncu rc=$?"
python tools/ncu_summary.py $O/full_$W.ncu-rep --out $O/${TAG}_${W}_full.md > /dev/null 2>&1
python tools/sass_mix.py $O/full_$W.ncu-rep --top 30 > $O/${TAG}_${W}_sass_mix.txt 2>&1
python tools/hotlines.py $O/full_$W.ncu-rep > $O/${TAG}_${W}_hot.txt 2>&1
rm -f $O/full_$W.ncu-rep
