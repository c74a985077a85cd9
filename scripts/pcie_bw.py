"""Host<->device copy bandwidth from pinned memory (the floor of bench.py's e2e leg): one stream vs
several concurrent streams, H2D alone and H2D with a concurrent D2H."""
import json, torch
nbytes = 2189721600
h = torch.empty(nbytes, dtype=torch.uint8).pin_memory()
d = torch.empty(nbytes, dtype=torch.uint8, device="cuda")
ho = torch.empty(nbytes // 3, dtype=torch.uint8).pin_memory()
do = torch.empty(nbytes // 3, dtype=torch.uint8, device="cuda")
def run(nstreams, with_d2h=False, reps=3):
    ss = [torch.cuda.Stream() for _ in range(nstreams)]
    sd = torch.cuda.Stream()
    chunk = nbytes // nstreams
    best = 1e9
    for _ in range(reps):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for s in ss + [sd]:
            s.wait_stream(torch.cuda.current_stream())
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        if with_d2h:
            with torch.cuda.stream(sd):
                ho.copy_(do, non_blocking=True)
        for s in ss + [sd]:
            torch.cuda.current_stream().wait_stream(s)
        e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    return best
for n in (1, 2, 4):
    for dd in (False, True):
        ms = run(n, dd)
        print(json.dumps({"h2d_streams": n, "concurrent_d2h": dd, "ms": round(ms, 2), "h2d_GBps": round(nbytes / ms / 1e6, 1)}))
