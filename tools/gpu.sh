#!/bin/bash
# Build locally (abort on failure), then run a command on the B200 box.
# usage: tools/gpu.sh TIMEOUT 'command'
set -e
cd "$(dirname "$0")/.."
python -m paracut_b200.build > /dev/null
timeout $(( $1 + 1200 )) /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
