import sys, time, ctypes, torch
sys.path.insert(0, ".")
import paper_2605_24840_b200 as nsr, workloads
p = workloads.cfg0_controlled(0)
H = torch.from_numpy(p.H).cuda(); R = torch.empty_like(H)
ws = nsr.alloc_workspace(nsr.ns_workspace_bytes(p.d), H.device)
lib = nsr.load_library()
for _ in range(20): nsr.ns_reflector(H, p.s, p.alpha, p.k, 100, 1e-12, R=R, ws=ws)
torch.cuda.synchronize()
n = 2000
t0 = time.perf_counter()
for _ in range(n): nsr.ns_reflector(H, p.s, p.alpha, p.k, 100, 1e-12, R=R, ws=ws)
t1 = time.perf_counter()
res = nsr.NsResult()
args = (ctypes.c_void_p(H.data_ptr()), 64, 64, float(p.s), float(p.alpha), int(p.k), 100, 1e-12, 0, 0,
        ctypes.c_void_p(R.data_ptr()), 64, ctypes.c_void_p(ws.data_ptr()), ws.numel(), ctypes.c_void_p(0), ctypes.byref(res))
t2 = time.perf_counter()
for _ in range(n): lib.ns_reflector(*args)
t3 = time.perf_counter()
s = torch.cuda.current_stream()
t4 = time.perf_counter()
for _ in range(n): torch.cuda.current_stream().cuda_stream
t5 = time.perf_counter()
print(f"python wrapper {1e6*(t1-t0)/n:.1f} us, raw ctypes {1e6*(t3-t2)/n:.1f} us, current_stream {1e6*(t5-t4)/n:.2f} us")
