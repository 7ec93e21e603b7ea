"""Per-CTA timeline of the step kernels (diagnostics).

Build the trace variant, then run on the GPU box:
    python -m paper_2007_06048_b200.build --variant trc -D MM_TRACE
    MM_LIB_VARIANT=trc python tools/step_trace.py 240 [name=value,...]
Prints, per step, each kernel's CTA start / end times (min/median/max, us
from the previous step's boundary-kernel end).  The MM_TRACE kernels write
(kernel, SM, start, end) with %globaltimer into a device ring that
mm_trace_dump reads; a normal build compiles it out.
"""
import sys, os, ctypes as C
os.environ.setdefault("CUDA_DEVICE_MAX_CONNECTIONS", "32")
sys.path.insert(0, '/root/repo')
import numpy as np
import paper_2007_06048_b200 as mm
from paper_2007_06048_b200 import _lib
g = int(sys.argv[1]); steps = 4
kv = dict(x.split('=') for x in sys.argv[2].split(',') if x) if len(sys.argv) > 2 else {}
_lib.reset_tuning()
for k, v in kv.items(): _lib.set_tuning(k, int(v))
n = (g, g, g)
grid = mm.make_grid(n, (20.0, 20.0, 20.0))
model = mm.default_layered_model(grid)
dt = mm.cfl_dt(model, grid, 0.8)
w = mm.ricker(25.0, dt, 40).samples
e = mm.AcousticCdEngine(grid, (0, 0, 0), n, model.vp, mm.EngineOptions(ndamping=(27,)*3, taper=True), dt, model.vmax)
e.run(w[:30], (g//2, g//2, g//2), record=False)
L = _lib.lib()
buf = (C.c_ulonglong * (4 * 65536))(); cnt = C.c_int()
L.mm_trace_dump(buf, 65536, C.byref(cnt))
e.run(w[30:30 + steps], (g//2, g//2, g//2), record=False)
L.mm_trace_dump(buf, 65536, C.byref(cnt))
a = np.frombuffer(buf, dtype=np.uint64)[:4 * cnt.value].reshape(-1, 4).astype(np.int64)
names={0:'p1z',1:'p1xy',2:'inner',3:'bnd'}
a=a[np.argsort(a[:,2])]
b=a[a[:,0]==3]
bs=b[np.argsort(b[:,2])]
per = int((a[:,0]==3).sum() // steps)
ends=[bs[i*per:(i+1)*per,3].max() for i in range(steps)]
for si in range(1, steps):
    lo=ends[si-1]; hi=ends[si]
    st=a[(a[:,2]>lo-2000)&(a[:,2]<=hi)]
    out=[]
    for k in range(4):
        ks=st[st[:,0]==k]
        if len(ks)==0: continue
        s_=np.sort((ks[:,2]-lo)/1e3); e_=np.sort((ks[:,3]-lo)/1e3)
        out.append(f"{names[k]} n{len(ks)} st {s_[0]:.0f}/{np.median(s_):.0f}/{s_[-1]:.0f} en {e_[0]:.0f}/{np.median(e_):.0f}/{e_[-1]:.0f}")
    print(f"{sys.argv[2] if len(sys.argv)>2 else 'default'} step {(hi-lo)/1e3:.1f}us | " + ' | '.join(out))
