#!/bin/bash
# Round profiling job (run under gpurun): default bench line (c5 + c3 secondary), the ncu
# launch list of the same command, per-config launch lists, CUPTI timelines, and one
# `--set full` capture of the top kernels of c5, c1 and c3.
#   bash tools/profile_round.sh r02
set -u
R=${1:-r02}
O=gpurun_out/prof
mkdir -p $O
python bench.py > $O/${R}_bench.json 2> $O/${R}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 6000 --csv \
    --log-file $O/${R}_c5_launches.csv python bench.py --steps 20 --warmup 3 --secondary '' --no-sweep --no-cpu-baseline \
    > /dev/null 2>&1
for c in c1 c2 c3 c4; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
        --log-file $O/${R}_${c}_launches.csv python bench.py --workload $c --secondary '' --no-sweep \
        --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
done
for c in c1 c2 c3 c4 c5; do
    timeout 300 python tools/cupti_timeline.py $c 3 > $O/${R}_${c}_timeline.txt 2>&1
done
# full sections for the top kernels (after warm-up launches)
timeout 900 ncu --set full --import-source on -k regex:"k_pencil_lane|k_fgemm|k_resfold|k_dft_fused|k_kr_combine|k_window|k_profiles" \
    -s 60 -c 12 -o $O/${R}_c5_full python bench.py --workload c5 --secondary '' --no-sweep --steps 3 --warmup 3 \
    --no-cpu-baseline > $O/${R}_c5_full.log 2>&1
timeout 900 ncu --set full --import-source on -k regex:"k_pencil|k_l0|k_triv_gemm|k_hankel|k_window|k_fill" \
    -s 40 -c 8 -o $O/${R}_c1_full python bench.py --workload c1 --secondary '' --no-sweep --steps 3 --warmup 3 \
    --no-cpu-baseline > $O/${R}_c1_full.log 2>&1
timeout 900 ncu --set full --import-source on -k regex:"k_sytrd|k_tridiag_eig3|k_hankel|k_dgemm|k_potf|k_window" \
    -s 40 -c 12 -o $O/${R}_c3_full python bench.py --workload c3 --secondary '' --no-sweep --steps 3 --warmup 3 \
    --no-cpu-baseline > $O/${R}_c3_full.log 2>&1
# c3 outside the Cholesky chain: lattice sum, contraction, tridiagonalisation, eigenvalues
timeout 900 ncu --set full --import-source on -k regex:"k_hankel|k_window_sum_staged|k_sytrd|k_tridiag_eig3|k_master|k_vgemm|k_triv_gemm" \
    -s 24 -c 8 -o $O/${R}_c3b_full python bench.py --workload c3 --secondary '' --no-sweep --steps 3 --warmup 3 \
    --no-cpu-baseline > $O/${R}_c3b_full.log 2>&1
ls -la $O
