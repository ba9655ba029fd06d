#!/bin/bash
# Developer pass: build, selected GPU tests (K=pytest -k expression), then tools/gpu_ab.sh
O=gpurun_out/${TAG:-t}
mkdir -p $O
python -c "import __graft_entry__ as g; g.build()" > $O/build.log 2>&1 || { tail -30 $O/build.log; exit 1; }
timeout 600 python -m pytest tests -m gpu -x -q -k "$K" > $O/pytest_k.log 2>&1; echo "pytest -k rc=$?"; tail -n 5 $O/pytest_k.log
NO_TEST=1 bash tools/gpu_ab.sh
