# One full round-end measurement on the GPU box (run from the repo root under gpurun):
#   tests, smoke, every bench config, the reference arm, ncu captures.
#   usage: bash tools/gpu_round.sh <tag>
cd $GRAFT_REPO_ROOT; mkdir -p gpurun_out
T=${1:-f}
timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pytest_$T.log 2>&1; echo rc=$? >> gpurun_out/pytest_$T.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$T.log 2>&1; echo rc=$? >> gpurun_out/smoke_$T.log
timeout 400 python bench.py > gpurun_out/bench_c2_$T.log 2>&1
for w in c1 c3 c4 c5; do timeout 300 python bench.py --workload $w > gpurun_out/bench_${w}_$T.log 2>&1; done
for w in c2 c3 c4 c5; do timeout 300 python bench.py --workload $w --data correlated --no-cpu-baseline > gpurun_out/bench_${w}corr_$T.log 2>&1; done
timeout 400 python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/bench_ref_c2_$T.log 2>&1
timeout 400 python bench.py --impl reference --workload c4 --steps 3 --warmup 3 > gpurun_out/bench_ref_c4_$T.log 2>&1
bash tools/gpu_profiles.sh $T
