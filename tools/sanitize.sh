#!/bin/bash
# compute-sanitizer memcheck + racecheck (+ synccheck) of the solve path on c1, c2, c3 (GPU box).
#   bash tools/sanitize.sh  ->  gpurun_out/sanitize_*.log
set -u
mkdir -p gpurun_out
CS=/usr/local/cuda/bin/compute-sanitizer
for tool in memcheck racecheck synccheck; do
    for c in c1 c2 c3; do
        timeout 900 $CS --tool $tool --error-exitcode 9 --print-limit 20 python tools/sanitize_solve.py $c \
            > gpurun_out/sanitize_${tool}_${c}.log 2>&1
        echo "$tool $c rc=$? $(grep -E 'ERROR SUMMARY|RACECHECK SUMMARY' gpurun_out/sanitize_${tool}_${c}.log | tail -1)"
    done
done
