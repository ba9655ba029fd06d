# usage: bash tools/ncu_exp.sh <config[@HxW]> <out tag> [kernel regex] -- ncu --set full of one launch (tools/exp.py), summarised
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/$2
timeout 600 ncu --set full --clock-control none --import-source on -k regex:${3:-fcfs} -s 2 -c 1 -o gpurun_out/$2/rep -f python tools/exp.py $1 --reps 1 > gpurun_out/$2/log 2>&1
python tools/sass_mix.py gpurun_out/$2/rep.ncu-rep --top 24 > gpurun_out/$2/mix.txt 2>&1
python tools/ncu_summary.py gpurun_out/$2/rep.ncu-rep --out gpurun_out/$2/sum.md > /dev/null 2>&1
ncu -i gpurun_out/$2/rep.ncu-rep --page source --csv > gpurun_out/$2/src.csv 2>/dev/null
rm -f gpurun_out/$2/rep.ncu-rep
