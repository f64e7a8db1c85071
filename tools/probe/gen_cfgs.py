"""Dev probe helper: write the five BASELINE configs as raw float32 files."""
import sys, numpy as np
out = sys.argv[1]
def cfg(k):
    if k == 1: r = np.random.default_rng(0); return r.standard_normal(1024)
    if k == 2:
        r = np.random.default_rng(1); n = 16384; c = r.random(n) < 0.5; z = r.standard_normal(n)
        return np.where(c, -2 + 0.5 * z, 2 + 1.0 * z)
    if k == 3:
        r = np.random.default_rng(2); n = 131072; c = r.random(n) < 0.7; u = r.random(n); e = r.exponential(0.5, n)
        return np.where(c, u, e)
    if k == 4: r = np.random.default_rng(3); return 3 + 2 * r.standard_normal(1048576)
    if k == 5:
        r = np.random.default_rng(4); n = 4194304; mu = np.array([-4, -1, 0, 2, 5.]); sd = np.array([.3, 1, .5, .8, 2])
        c = r.integers(0, 5, n); z = r.standard_normal(n); return mu[c] + sd[c] * z
for k in range(1, 6):
    cfg(k).astype(np.float32).tofile(f"{out}/cfg{k}.f32")
# adversarial extras (same recipes as paper_1505_02100_b200/inputs.py)
r = np.random.default_rng(4); (np.round(r.standard_normal(12000) * 37 / 6.0) * (6.0 / 37)).astype(np.float32).tofile(f"{out}/ties.f32")
r = np.random.default_rng(5); (1.0e6 + r.standard_normal(12000)).astype(np.float32).tofile(f"{out}/offset.f32")
