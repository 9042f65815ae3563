#!/usr/bin/env bash
# the round-2 part of tools/sanitize.sh only
out=${1:-gpurun_out/sanitize_r02}
mkdir -p "$out"
CS=/usr/local/cuda/bin/compute-sanitizer
sed -n '/^# round 2/,$p' tools/sanitize.sh > /tmp/san_r02.sh
out="$out" CS="$CS" bash -c "out=$out; CS=$CS; source /tmp/san_r02.sh"
