#!/bin/bash
O=gpurun_out/${TAG:-bm}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
FCFS_PLANE_BM=1 timeout 600 python -m pytest tests -m gpu -x -q -k "plane and not plane3" > $O/pytest_bm.log 2>&1; echo "pytest bm rc=$?"; tail -n 3 $O/pytest_bm.log
NO_TEST=1 bash tools/gpu_ab.sh
[ -n "$FULL" ] && { timeout 900 python -m pytest tests -m gpu -x -q > $O/pytest_gpu.log 2>&1; echo "pytest gpu rc=$?"; tail -n 3 $O/pytest_gpu.log; }
