import time, ctypes, numpy as np, torch
x = torch.randn(10000*3584, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
def t(f, name):
    torch.cuda.synchronize(); s=time.perf_counter(); r=f(); torch.cuda.synchronize(); print(name, round((time.perf_counter()-s)*1e3,1), "ms"); return r
for _ in range(2):
    t(lambda: x.cpu(), "x.cpu()")
    t(lambda: x.to("cpu"), "to cpu")
    h = np.empty(x.numel())
    t(lambda: torch.from_numpy(h).copy_(x), "copy_ into numpy")
    cudart = ctypes.CDLL("libcudart.so.12") if False else None
    p = t(lambda: torch.empty(x.numel(), dtype=torch.float64, pin_memory=True), "pinned alloc")
    t(lambda: p.copy_(x), "copy to pinned")
    t(lambda: np.array(p.numpy()), "host memcpy from pinned")
    hh = np.empty(x.numel())
    t(lambda: torch.cuda.cudart().cudaHostRegister(hh.ctypes.data, hh.nbytes, 0), "hostRegister")
    t(lambda: torch.from_numpy(hh).copy_(x), "copy into registered")
    torch.cuda.cudart().cudaHostUnregister(hh.ctypes.data)
    v = np.random.rand(x.numel())
    t(lambda: torch.from_numpy(v).to("cuda"), "H2D pageable")
