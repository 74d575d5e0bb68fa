#!/bin/bash
# usage: tools/gpu.sh LOGFILE TIMEOUT 'command'   -- rebuild libautosp.so, then run on a B200
cd /root/repo || exit 1
python paper_2604_27089_b200/_build.py > /dev/null || { echo "BUILD FAILED" > "$1"; exit 1; }
timeout $(( $2 + 600 )) /usr/local/graft/bin/gpurun --timeout "$2" -- "$3" > "$1" 2>&1
