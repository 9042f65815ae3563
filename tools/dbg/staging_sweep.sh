#!/usr/bin/env bash
# pageable e2e at C2 over staging chunk / ring / NT / thread settings
out=gpurun_out/${1:-staging}
mkdir -p $out
for cfg in "32768 4 1 8" "32768 4 0 8" "4096 8 0 8" "4096 8 1 8" "2048 16 0 8" "8192 8 0 8" "4096 8 0 6" "4096 8 0 4"; do
  set -- $cfg
  COLOC_STAGING_CHUNK_KB=$1 COLOC_STAGING_RING=$2 COLOC_STAGING_H2D_NT=$3 COLOC_STAGING_THREADS=$4 \
    timeout 300 python tools/dbg/pageable_e2e.py $((1<<30)) 4 2 >> $out/sweep.jsonl 2>&1
done
