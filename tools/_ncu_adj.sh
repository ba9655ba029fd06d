python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/n7
timeout 600 ncu --set full --clock-control none --import-source on -k regex:adjoint_tile -s 0 -c 1 -o gpurun_out/n7/band -f python tools/exp.py C3B --reps 1 > gpurun_out/n7/log 2>&1
python tools/sass_mix.py gpurun_out/n7/band.ncu-rep --top 16 > gpurun_out/n7/mix.txt 2>&1
python tools/ncu_summary.py gpurun_out/n7/band.ncu-rep --out gpurun_out/n7/sum.md > /dev/null 2>&1
ncu -i gpurun_out/n7/band.ncu-rep --page source --csv > gpurun_out/n7/src.csv 2>/dev/null
rm -f gpurun_out/n7/band.ncu-rep
