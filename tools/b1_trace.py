# In-graph timeline of one batch-1 decode (MTG_TRACE=1): per step kernel,
# the gap after the previous kernel's last CTA and the kernel's duration.
import os, sys
os.environ.setdefault("MTG_TRACE", "1")  # 2: also per-phase times
sys.path.insert(0, '/root/repo')
import paper_2008_04885_b200 as mt
from bench import CONFIG_20_2, sources
for name in sys.argv[1:] or ["int8", "f32"]:
    prec = {'f32': mt.F32, 'int8': mt.INT8, 'bf16': mt.BF16}[name]
    m = mt.Model.create(CONFIG_20_2, seed=1, precision=prec)
    cfg = mt.BeamConfig(5, 0, 1.0)
    m.stage(sources(1, 7)); m.run_staged(cfg); m.run_staged(cfg)
    print(name); print(m.diag_report())
