"""How fast does a CUDA graph dispatch many tiny kernels spread over S streams?
(attribution of the non-edge part of the step: launch-rate vs work)"""
import torch, time
torch.cuda.init()
for S, K in ((1, 2600), (16, 2600), (32, 2600), (16, 1300)):
    xs = [torch.zeros(1024, device="cuda") for _ in range(S)]
    streams = [torch.cuda.Stream() for _ in range(S)]
    g = torch.cuda.CUDAGraph()
    root = torch.cuda.Stream()
    with torch.cuda.stream(root):
        g.capture_begin()
        ev0 = torch.cuda.Event(); ev0.record(root)
        for i, st in enumerate(streams):
            st.wait_event(ev0)
            with torch.cuda.stream(st):
                for _ in range(K // S):
                    xs[i].add_(1.0)
        for st in streams:
            e = torch.cuda.Event(); e.record(st); root.wait_event(e)
        g.capture_end()
    for _ in range(3): g.replay()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record(); 
    for _ in range(10): g.replay()
    b.record(); torch.cuda.synchronize()
    print(f"streams={S} kernels={K}: {a.elapsed_time(b)/10:.3f} ms per graph, {a.elapsed_time(b)/10/K*1000:.2f} us/kernel", flush=True)
