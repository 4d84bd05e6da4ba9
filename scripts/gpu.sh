#!/bin/bash
# Build the in-tree library here (so the snapshot carries an up-to-date .so), then run the
# given command on a B200 through gpurun.  Usage: scripts/gpu.sh <timeout_s> '<command>'
set -e
cd "$(dirname "$0")/.."
python paper_1409_2556_b200/build.py > /dev/null
exec /usr/local/graft/bin/gpurun --timeout "$1" -- "$2"
