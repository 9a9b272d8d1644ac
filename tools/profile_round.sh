#!/bin/bash
# Round profiling job (run under gpurun): default bench line, the ncu launch list of the
# same command, per-config launch lists, and one `--set full` capture of the top kernels.
#   bash tools/profile_round.sh r01
set -u
R=${1:-r01}
mkdir -p gpurun_out/prof
python bench.py > gpurun_out/prof/${R}_bench.json 2> gpurun_out/prof/${R}_bench.err
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none -c 4000 --csv \
    --log-file gpurun_out/prof/${R}_c2_launches.csv python bench.py > /dev/null 2>&1
for c in c1 c3 c4 c5; do
    timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none -c 2000 --csv \
        --log-file gpurun_out/prof/${R}_${c}_launches.csv python bench.py --workload $c --steps 3 --warmup 3 \
        --no-cpu-baseline > /dev/null 2>&1
done
# full sections for the top kernels of the default workload (after warm-up launches)
timeout 900 ncu --set full --import-source on -k regex:"k_pencil|k_l0_scan|k_l0_sample|k_triv_gemm|k_resfold|k_dft_axis2|k_fill|k_master|k_window" \
    -s 40 -c 14 -o gpurun_out/prof/${R}_c2_full python bench.py --workload c2 --steps 3 --warmup 3 \
    --no-cpu-baseline > gpurun_out/prof/${R}_c2_full.log 2>&1
timeout 900 ncu --set full --import-source on -k regex:"k_pencil|k_resfold|k_triv_gemm|k_window|k_l0_scan" \
    -s 30 -c 8 -o gpurun_out/prof/${R}_c4_full python bench.py --workload c4 --steps 3 --warmup 3 \
    --no-cpu-baseline > gpurun_out/prof/${R}_c4_full.log 2>&1
timeout 900 ncu --set full --import-source on -k regex:"k_sytrd|k_tridiag_eig3|k_trtri_leaf|k_hankel" \
    -s 8 -c 4 -o gpurun_out/prof/${R}_c3_full python bench.py --workload c3 --steps 3 --warmup 3 \
    --no-cpu-baseline > gpurun_out/prof/${R}_c3_full.log 2>&1
timeout 600 python tools/table1.py > gpurun_out/prof/${R}_table1.json 2> gpurun_out/prof/${R}_table1.err
ls -la gpurun_out/prof
