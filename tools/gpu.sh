#!/bin/bash
# Rebuild in-tree (library + oracle) and run a command on the B200 box via gpurun.
# usage: tools/gpu.sh TIMEOUT 'command'
set -e
cd /root/repo
python -c "import __graft_entry__ as g; g.build()"
T=${1:-900}; shift
exec timeout $((T + 1500)) /usr/local/graft/bin/gpurun --timeout $T -- "$@"
