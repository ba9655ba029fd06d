# ncu --set full of one tiled-kernel launch of tools/tiled_bench.py (27/11 bilinear), summarised under gpurun_out/t1
python -c "import __graft_entry__ as g; g.build()" > /dev/null 2>&1
mkdir -p gpurun_out/t1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:tile -s 3 -c 1 -o gpurun_out/t1/rep -f python tools/tiled_bench.py > gpurun_out/t1/log 2>&1
python tools/sass_mix.py gpurun_out/t1/rep.ncu-rep --top 24 > gpurun_out/t1/mix.txt 2>&1
python tools/ncu_summary.py gpurun_out/t1/rep.ncu-rep --out gpurun_out/t1/sum.md > /dev/null 2>&1
rm -f gpurun_out/t1/rep.ncu-rep
