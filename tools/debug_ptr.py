import torch, numpy as np
x = np.zeros(100)
t = torch.zeros(10, dtype=torch.float64, device="cuda")
p = torch.zeros(10, dtype=torch.float64).pin_memory()
try:
    from cuda.bindings import runtime as cr
except Exception:
    from cuda import cudart as cr
for name, ptr in (("pageable", x.ctypes.data), ("device", t.data_ptr()), ("pinned", p.data_ptr())):
    err, attr = cr.cudaPointerGetAttributes(ptr)
    print(name, err, attr.type, attr.devicePointer, attr.hostPointer)
