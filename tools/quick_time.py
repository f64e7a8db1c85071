"""Dev helper: time plugin_h and each psi pass on a BASELINE config (CUDA events)."""
import sys, os, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1505_02100_b200 import inputs, plugin as P
k = int(sys.argv[1]) if len(sys.argv) > 1 else 4
reps = int(sys.argv[2]) if len(sys.argv) > 2 else 3
x = torch.from_numpy(inputs.config_data(k)).cuda()
n = x.numel()
ws = P.workspace(n); out = P.new_result()
for _ in range(2): P.plugin_h(x, out, ws)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
ts = []
for _ in range(reps):
    e0.record(); P.plugin_h(x, out, ws); e1.record(); torch.cuda.synchronize(); ts.append(e0.elapsed_time(e1))
r = P.read_result(out)
pairs = n * (n - 1) / 2
t = min(ts) / 1e3
print(f"cfg{k} n={n} plugin_h min {min(ts):.3f} ms  -> {2*pairs/t/1e9:.1f} GPairs/s (both passes) ; per SM-clk @1.965GHz: {2*pairs/t/148/1.965e9:.2f}")
print({k2: r[k2] for k2 in ('status','h','psi6_z','psi4_z','g1','g2')})
