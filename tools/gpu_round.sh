#!/bin/bash
# One GPU-box pass: gpu tests, smoke, bench lines for every workload, ncu launch
# lists of the bench commands, ncu --set full of the dominant kernels.
# Usage (from the repo root, on the box): bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; tail -30 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?" ; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
[ -n "$ONLY_FULL" ] && { NO_BENCH=1; }
if [ -z "$NO_BENCH" ]; then
timeout 900 python bench.py > $O/bench_default.json 2> $O/bench_default.err; echo "bench default rc=$?"
for w in ${WL:-C2 C3 C4 C5 A1 A2 V1 V2 C3B C3W}; do
  timeout 600 python bench.py --workload $w --no-cpu-baseline > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?"
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $O/bench_reference.json 2> $O/bench_reference.err; echo "bench reference rc=$?"
fi
for w in ${NW:-C2 C3 C4 C5 A1 V1 V2 C3B C3W}; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$w.csv \
  python bench.py --workload $w --steps 2 --warmup 3 --soak-s 0 --no-e2e --no-cpu-baseline > $O/ncu_launch_$w.log 2>&1; echo "ncu launches $w rc=$?"
done
[ -n "$NO_FULL" ] && exit 0
for w in ${NW:-C2 C3 C4 C5 A1 V1 V2 C3B C3W}; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fcfs -s 4 -c 2 -o $O/full_$w -f \
  python bench.py --workload $w --steps 2 --warmup 3 --soak-s 0 --no-e2e --no-cpu-baseline > $O/ncu_full_$w.log 2>&1; echo "ncu full $w rc=$?"
  # summaries on the box (raw reports exceed the copy-back limit); keep the SASS mix too
  key=$w; match=""; [ "$w" = "C2" ] && key="C2a+C2b"; [ "$w" = "C4" ] && { key="C4a"; match="7, 5, 7, 5"; }
  python tools/ncu_summary.py $O/full_$w.ncu-rep --out $O/${TAG}_${w}_full.md --traffic-key "$key" \
    ${match:+--traffic-match "$match"} > /dev/null 2>&1
  cp profiles/traffic.json $O/traffic.json 2>/dev/null
  python tools/sass_mix.py $O/full_$w.ncu-rep --top 30 > $O/${TAG}_${w}_sass_mix.txt 2>&1
  [ -z "$KEEP_REP" ] && rm -f $O/full_$w.ncu-rep
done
