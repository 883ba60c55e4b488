# ncu captures for profiles/: launch list of bench.py (c2), --set full of the pair
# kernel (device-resident and host-buffer mode) and of the multi-reference kernel (c3).
#   usage: bash tools/gpu_profiles.sh <tag>   (then: python tools/ncu_summary.py ...)
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${1:-p}
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_c2_$T.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --clock-window 0 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"bleu_pair" -s 70 -c 1 -o gpurun_out/prof_pair_c2_$T python bench.py --steps 3 --warmup 3 --no-cpu-baseline --clock-window 0 > gpurun_out/ncu_pair_c2_$T.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"bleu_pair" -s 3 -c 1 -o gpurun_out/prof_pair_host_$T python tools/e2e_only.py c2 > gpurun_out/ncu_pair_host_$T.log 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"bleu_multi" -s 40 -c 1 -o gpurun_out/prof_multi_c3_$T python bench.py --workload c3 --steps 3 --warmup 3 --no-cpu-baseline --clock-window 0 > gpurun_out/ncu_multi_c3_$T.log 2>&1
