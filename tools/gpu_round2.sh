# Round-2 measurement on the GPU box (run from the repo root under gpurun):
#   tests, smoke, the default bench line (+ configs), the reference arm,
#   ncu launch list + --set full captures + DRAM bytes of every config,
#   compute-sanitizer on the new kernels.   usage: bash tools/gpu_round2.sh <tag>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${1:-r02}
timeout 1500 python -m pytest tests -m gpu -q > gpurun_out/${T}_pytest_gpu.log 2>&1; echo rc=$? >> gpurun_out/${T}_pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/${T}_smoke.log 2>&1; echo rc=$? >> gpurun_out/${T}_smoke.log
timeout 900 python bench.py > gpurun_out/${T}_bench_c2.json.log 2>&1
timeout 600 python bench.py --impl reference --steps 5 --warmup 3 > gpurun_out/${T}_bench_ref_c2.json.log 2>&1
timeout 600 python bench.py --impl reference --workload c4 --steps 3 --warmup 3 > gpurun_out/${T}_bench_ref_c4.json.log 2>&1
timeout 600 python bench.py --impl reference --workload c5 --steps 2 --warmup 3 > gpurun_out/${T}_bench_ref_c5.json.log 2>&1
timeout 400 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/${T}_launches_c2.csv python bench.py --steps 20 --warmup 3 --no-cpu-baseline --no-configs --clock-window 0 > /dev/null 2>&1
M=gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum
for wd in "c1 uniform" "c2 uniform" "c2 correlated" "c2 zipf" "c2 vocab1" "c3 uniform" "c3 correlated" "c4 uniform" "c4 correlated" "c5 uniform" "c5 correlated"; do
  set -- $wd
  timeout 300 ncu --metrics $M --clock-control none --csv --log-file gpurun_out/${T}_dram_$1_$2.csv python tools/kernel_times.py $1 $2 1 > /dev/null 2>&1
done
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"bleu_pair" -c 1 -o gpurun_out/${T}_prof_pair_c2 python tools/kernel_times.py c2 uniform 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"bleu_pair" -c 1 -o gpurun_out/${T}_prof_pair_c2corr python tools/kernel_times.py c2 correlated 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"bleu_pair" -c 1 -o gpurun_out/${T}_prof_pair_c4 python tools/kernel_times.py c4 uniform 1 > /dev/null 2>&1
timeout 400 ncu --set full --clock-control none --import-source on -k regex:"bleu_multi" -c 1 -o gpurun_out/${T}_prof_multi_c3 python tools/kernel_times.py c3 uniform 1 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:"bleu_sparse" -c 1 -o gpurun_out/${T}_prof_sparse_c5 python tools/kernel_times.py c5 uniform 1 > /dev/null 2>&1
(
timeout 600 compute-sanitizer --tool memcheck python tools/kernel_times.py c2 correlated 1
TB_FORCE_SPARSE=1 timeout 600 compute-sanitizer --tool memcheck python tools/kernel_times.py c2 uniform 1
TB_FORCE_SPARSE=1 timeout 600 compute-sanitizer --tool memcheck python tools/kernel_times.py c3 correlated 1
TB_FORCE_SPARSE=1 timeout 600 compute-sanitizer --tool synccheck python tools/kernel_times.py c2 uniform 1
TB_FORCE_SPARSE=1 timeout 600 compute-sanitizer --tool initcheck python tools/kernel_times.py c1 uniform 1
TB_FORCE_SPARSE=1 timeout 600 compute-sanitizer --tool racecheck python tools/kernel_times.py c1 uniform 1
timeout 600 compute-sanitizer --tool memcheck python -m pytest -q -x tests/test_plugin_gpu.py -k "unique or flatten" -p no:cacheprovider
timeout 600 compute-sanitizer --tool racecheck python -m pytest -q -x tests/test_plugin_gpu.py -k "golden" -p no:cacheprovider
) > gpurun_out/${T}_sanitizers.log 2>&1
echo done
