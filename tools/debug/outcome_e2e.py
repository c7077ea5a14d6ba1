"""Break down the outcome-record e2e at n = 14: H2D alone vs histogram + stage per chunk."""
import sys, time, torch
sys.path.insert(0, "/root/repo")
import paper_1602_08604_b200 as lre
from paper_1602_08604_b200.simulate import generate_device_outcomes

n, shots = int(sys.argv[1]) if len(sys.argv) > 1 else 14, 1000
chunk = int(sys.argv[2]) if len(sys.argv) > 2 else 65610
st = lre.StateDescriptor("ghz", n)
rows = 3**n
host = []
for lo in range(0, rows, chunk):
    hi = min(rows, lo + chunk)
    o = generate_device_outcomes(st, shots, seed=1, w_begin=lo, w_end=hi)
    h = torch.empty(tuple(o.shape), dtype=torch.uint16, pin_memory=True); h.copy_(o); host.append((lo, hi, h))
del o
plan = lre.LREPlan(n, shots)
dev = torch.device("cuda")
comp = torch.cuda.current_stream(); copy = torch.cuda.Stream()
bufs = [torch.empty((chunk, shots), dtype=torch.uint16, device=dev) for _ in range(2)]
def run(do_h2d=True, do_gpu=True, validate=True):
    ev_c = [torch.cuda.Event() for _ in range(2)]; ev_u = [torch.cuda.Event() for _ in range(2)]
    torch.cuda.synchronize(); t = time.perf_counter()
    for k, (lo, hi, h) in enumerate(host):
        b = k % 2
        copy.wait_event(ev_u[b])
        with torch.cuda.stream(copy):
            if do_h2d: bufs[b][: hi - lo].copy_(h, non_blocking=True)
            ev_c[b].record(copy)
        comp.wait_event(ev_c[b])
        if do_gpu: plan.stage_outcomes(bufs[b][: hi - lo], lo, hi, comp, validate=validate)
        ev_u[b].record(comp)
    torch.cuda.synchronize(); dt = time.perf_counter() - t
    plan._checks = []
    return dt
run()
print("full", run()); print("h2d only", run(do_gpu=False)); print("gpu only", run(do_h2d=False)); print("no validate", run(validate=False))
