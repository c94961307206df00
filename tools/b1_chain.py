# In-graph cost of each small-batch (batch-1) decode-step kernel: the kernel
# chained N times inside one CUDA graph with PDL (mtg_time_kernel ids 10-15).
import ctypes, sys
sys.path.insert(0, '/root/repo')
import paper_2008_04885_b200 as mt
from bench import CONFIG_20_2, sources
NAMES = {10: "noop (PDL floor)", 11: "gemv wo (+res)", 12: "gemv w1 (+LN,b1,relu)",
         13: "gemv logits (+LN, partials)", 14: "self attention (t=56)", 15: "softmax/top-k merge",
         16: "small self attention (t=56)", 17: "small cross attention"}
for name in sys.argv[1:] or ["int8", "f32", "bf16"]:
    prec = {'f32': mt.F32, 'int8': mt.INT8, 'bf16': mt.BF16}[name]
    m = mt.Model.create(CONFIG_20_2, seed=1, precision=prec)
    m.stage(sources(1, 7)); m.run_staged(mt.BeamConfig(5, 0, 1.0))
    out = []
    for kid, label in NAMES.items():
        ms, by, fl = ctypes.c_float(), ctypes.c_double(), ctypes.c_double()
        rc = mt.lib().mtg_time_kernel(m._h, kid, 200, ctypes.byref(ms), ctypes.byref(by), ctypes.byref(fl))
        out.append(f"  {label:30s} {1000 * ms.value:7.2f} us" + (f"  {by.value / ms.value / 1e6:8.1f} GB/s" if rc == 0 and by.value else "") if rc == 0 else f"  {label}: rc={rc} {mt.lib().mtg_last_error().decode()}")
    print(name); print("\n".join(out))
