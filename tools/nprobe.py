import sys, time, torch
sys.path.insert(0, '/root/repo')
import paper_2008_04885_b200 as mt
from tools.sweep import BASE, srcs, timed
prec = {'f32': mt.F32, 'int8': mt.INT8}[sys.argv[1]]
m = mt.Model.create(dict(BASE, num_encoder_layers=20, num_decoder_layers=2), seed=1, precision=prec)
bc = mt.BeamConfig(5, 0, 1.0)
for L in (20, 40, 60):
    line = f"len {L}:"
    for n in (64, 128, 192, 256):
        m.stage(srcs(n, L, 7)); t = timed(lambda: m.run_staged(bc))
        line += f"  n{n} {n / t:.0f}/s"
    print(line, flush=True)
