#!/bin/bash
# build locally, stop on a compile error, else run the given command on the GPU box
cd /root/repo
python paper_2203_10670_b200/build.py > /tmp/b.log 2>&1
if grep -q "error" /tmp/b.log; then grep -A3 error /tmp/b.log | head -20; echo BUILD_ERR; exit 1; fi
timeout $(( ${GT:-1800} + 1200 )) /usr/local/graft/bin/gpurun --timeout ${GT:-1800} -- "$1" 2>&1 | tail -${TL:-12}
