"""Graph replay vs direct launches of the c2 step (GPU box): why bench.py times
plan.run() — replaying 64 alternating one-kernel CUDA graphs costs extra GPU
time per step at large step counts (profiles/r01_experiments.md)."""
import sys, time, torch
sys.path.insert(0, '/root/repo')
import bench, paper_2510_05485_b200 as tb
b, l, v, r, sm = bench.WORKLOADS["c2"][:5]
dev = torch.device("cuda", 0)
plans = []
gen = torch.Generator(device=dev)
for k in range(64):
    gen.manual_seed(k)
    def draw():
        return tb.TokenBatch.trusted(torch.randint(0, v, (b, l), generator=gen, device=dev, dtype=torch.int32),
                                     torch.randint(l // 2, l + 1, (b,), generator=gen, device=dev, dtype=torch.int64))
    plans.append(tb.SentenceBleuPlan(draw(), [draw()], tb.BleuConfig()))
for p in plans: p.capture()
for K in (20, 200, 1000, 20, 200):
    for k in range(200): plans[k % 64].replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t0 = time.perf_counter(); e0.record()
    for k in range(K): plans[k % 64].replay()
    e1.record(); t1 = time.perf_counter(); torch.cuda.synchronize()
    print(f"K={K}: gpu {e0.elapsed_time(e1)*1000/K:.2f} us/step, host enqueue {(t1-t0)*1e6/K:.2f} us/step")
# same plan repeatedly (L2 resident)
for K in (200,):
    torch.cuda.synchronize(); e0.record()
    for k in range(K): plans[0].replay()
    e1.record(); torch.cuda.synchronize()
    print(f"same batch K={K}: gpu {e0.elapsed_time(e1)*1000/K:.2f} us/step")
# raw run() without graphs
torch.cuda.synchronize(); t0=time.perf_counter(); e0.record()
for k in range(200): plans[k % 64].run()
e1.record(); t1=time.perf_counter(); torch.cuda.synchronize()
print(f"run() K=200: gpu {e0.elapsed_time(e1)*1000/200:.2f} us/step host {(t1-t0)*1e6/200:.2f}")
