#!/bin/bash
# A/B timing of engine variants (under gpurun): tools/_ab/<variant>/liblatham_b200.so are
# swapped into the package in turn, each timed R times alternately on the given workloads.
#   bash tools/ab.sh "A B C" "c5 c2" 3
set -u
VARS=${1:-"A B"}; WLS=${2:-c5}; R=${3:-3}
cp paper_1408_3839_b200/_lib/liblatham_b200.so /tmp/ab_keep.so
for r in $(seq 1 $R); do
  for v in $VARS; do
    cp tools/_ab/$v/liblatham_b200.so paper_1408_3839_b200/_lib/liblatham_b200.so
    for w in $WLS; do
      python bench.py --workload $w --secondary "" --no-sweep --no-cpu-baseline --steps 200 2>/dev/null | \
        python -c "import json,sys; d=json.loads(sys.stdin.read().strip().splitlines()[-1]); print('$v', '$w', round(d['value']*1000,1), round(d['e2e']['value']*1000,1))"
    done
  done
done | sort | awk '{k=$1" "$2; v[k]=v[k]" "$3"/"$4} END {for (k in v) print k":"v[k]}' | sort
cp /tmp/ab_keep.so paper_1408_3839_b200/_lib/liblatham_b200.so
