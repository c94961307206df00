import sys, torch
sys.path.insert(0, '/root/repo')
import paper_2008_04885_b200 as mt
from bench import CONFIG_20_2, sources
prec = {'f32': mt.F32, 'int8': mt.INT8, 'bf16': mt.BF16}[sys.argv[1] if len(sys.argv) > 1 else 'int8']
m = mt.Model.create(CONFIG_20_2, seed=1, precision=prec)
n = int(sys.argv[2]) if len(sys.argv) > 2 else 64
m.stage(sources(n, 7)); cfg = mt.BeamConfig(5, 0, 1.0)
m.run_staged(cfg); m.run_staged(cfg); torch.cuda.synchronize()
torch.cuda.profiler.start()
m.run_staged(cfg); torch.cuda.synchronize()
torch.cuda.profiler.stop()
print('launches', m.last_launch_count())
