cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
TAG=${1:-b}
timeout 400 python bench.py > gpurun_out/bench_default_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_default_$TAG.log
timeout 400 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/bench_ref_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/bench_ref_$TAG.log
nproc > gpurun_out/nproc_$TAG.txt
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --clock-window 0 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"bleu_(group|pair)" -s 70 -c 1 -o gpurun_out/prof_$TAG python bench.py --steps 3 --warmup 3 --no-cpu-baseline --clock-window 0 > gpurun_out/ncu_full_$TAG.log 2>&1
