#!/bin/bash
# B200-scale runs of the experiment harness (python -m paper_1209_3314_b200 bench)
# -> gpurun_out/experiments.txt
mkdir -p gpurun_out
{
for e in "queue 4096x4096" "coverage 4096x4096" "overflow 2048x2048" "scaling 4096x4096" "tilesize 8192x8192"; do
  set -- $e
  echo "## $1 $2"
  python -m paper_1209_3314_b200 bench --experiment $1 --size $2 --workers 4
done
} > gpurun_out/experiments.txt 2>&1
