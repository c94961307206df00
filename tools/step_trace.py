# In-graph timeline of one batched decode (MTG_TRACE=1): per step kernel, the
# gap after the previous traced kernel's last CTA and the kernel's duration
# (first post-wait CTA to last CTA exit), averaged over the steps.
#   python tools/step_trace.py <f32|int8|bf16> [sentences=64]
import os, sys
os.environ.setdefault("MTG_TRACE", "1")  # 2: also per-phase times
sys.path.insert(0, '/root/repo')
import paper_2008_04885_b200 as mt
from bench import CONFIG_20_2, sources
name = sys.argv[1] if len(sys.argv) > 1 else "f32"
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
prec = {'f32': mt.F32, 'int8': mt.INT8, 'bf16': mt.BF16}[name]
m = mt.Model.create(CONFIG_20_2, seed=1, precision=prec)
cfg = mt.BeamConfig(5, 0, 1.0)
m.stage(sources(n, 7)); m.run_staged(cfg); m.run_staged(cfg)
print(name, n); print(m.diag_report())
