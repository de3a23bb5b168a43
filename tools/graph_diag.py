import time, torch, sys
sys.path.insert(0,'/root/repo')
import paper_1711_00903_b200 as hx
from paper_1711_00903_b200 import cg
mesh = hx.build_cube_mesh(8, 2.0)
op = hx.make_operator(hx.BP35, 7, mesh, lam=0.0)
b = torch.randn(op.n_el, op.n_p, dtype=torch.float64, device="cuda")
st = cg._AssembledState(op, 8, b, True, None, None)
stream = cg._stream(op.device)
cg._assembled_setup(op, 8, b, st, stream)
w=st.w
def block():
    c=0
    strm=cg._stream(op.device)
    for _ in range(10):
        nx=cg._assembled_step(op, 8, st, c, strm, None)
        hx._native.lib().hx_cg_direction(hx._native.ptr(w.p), hx._native.ptr(w.r), b.numel(), hx._native.ptr(w.rr[nx]), hx._native.ptr(w.rr[c]), strm)
        c=nx
block(); torch.cuda.synchronize()
t=time.perf_counter(); block(); torch.cuda.synchronize(); print('eager block ms', (time.perf_counter()-t)*1e3)
t=time.perf_counter(); rep=cg._graphed(block); torch.cuda.synchronize(); print('capture ms', (time.perf_counter()-t)*1e3)
for i in range(3):
    t=time.perf_counter(); rep(); torch.cuda.synchronize(); print('replay ms', (time.perf_counter()-t)*1e3)
t=time.perf_counter()
for i in range(20): rep()
torch.cuda.synchronize(); print('20 replays ms', (time.perf_counter()-t)*1e3)
s,e=torch.cuda.Event(enable_timing=True),torch.cuda.Event(enable_timing=True)
s.record(); rep(); e.record(); e.synchronize(); print('replay gpu ms', s.elapsed_time(e))
s.record(); block(); e.record(); e.synchronize(); print('eager gpu ms', s.elapsed_time(e))
