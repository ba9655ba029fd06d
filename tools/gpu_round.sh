#!/bin/bash
# One GPU-box pass: gpu tests, smoke, bench lines for every workload, ncu launch
# list of the default bench command, ncu --set full of the dominant kernels.
# Usage (from the repo root, on the box): bash tools/gpu_round.sh [tag]
TAG=${1:-r01}
O=gpurun_out/$TAG
mkdir -p $O
nvidia-smi > $O/nvidia-smi.txt 2>&1
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { echo BUILD FAILED; tail -30 $O/build.log; exit 1; }
timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?" ; tail -3 $O/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo "smoke rc=$?"; tail -2 $O/smoke.log
for w in C2 C3 C4 C5; do
  timeout 600 python bench.py --workload $w --steps 100 --warmup 5 > $O/bench_$w.json 2> $O/bench_$w.err; echo "bench $w rc=$?"; cat $O/bench_$w.json | cut -c1-400
done
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_C2.csv \
  python bench.py --steps 2 --warmup 3 --soak-s 0 --no-e2e --no-cpu-baseline > $O/ncu_launch.log 2>&1; echo "ncu launches rc=$?"
for w in C3 C4 C5; do
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file $O/launches_$w.csv \
  python bench.py --workload $w --steps 2 --warmup 3 --soak-s 0 --no-e2e --no-cpu-baseline > $O/ncu_launch_$w.log 2>&1; echo "ncu launches $w rc=$?"
done
# full captures of one launch of each hot kernel (skip warm-up launches)
for w in C2 C3 C4 C5; do
timeout 900 ncu --set full --clock-control none --import-source on -k regex:fcfs -s 4 -c 2 -o $O/full_$w -f \
  python bench.py --workload $w --steps 2 --warmup 3 --soak-s 0 --no-e2e --no-cpu-baseline > $O/ncu_full_$w.log 2>&1; echo "ncu full $w rc=$?"
done
