import sys, time, os
sys.path.insert(0, '.')
import torch, paper_2510_09417_b200 as vq
xs, ys = vq.generate('square', 10**8, 2)
X, Y = torch.from_numpy(xs).cuda(), torch.from_numpy(ys).cuda()
out = torch.empty(10**8, dtype=torch.int32, device='cuda')
st = torch.cuda.current_stream()
for _ in range(5): vq.hull_device(X, Y, stream=st, out=out, u32=True)
torch.cuda.synchronize()
for label, fn in [('hull_device', lambda: vq.hull_device(X, Y, stream=st, out=out, u32=True)),
                  ('raw ctypes', None)]:
    if fn is None:
        import ctypes as C
        L = vq.lib(); cnt = C.c_uint64(); xp, yp, op, sp = X.data_ptr(), Y.data_ptr(), out.data_ptr(), st.cuda_stream
        fn = lambda: L.vqhull_cuda_hull_u32(xp, yp, 10**8, op, C.byref(cnt), sp)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(st); t0 = time.perf_counter()
    for _ in range(20): fn()
    e1.record(st); torch.cuda.synchronize()
    print(label, e0.elapsed_time(e1) / 20, (time.perf_counter() - t0) / 20 * 1e3)
