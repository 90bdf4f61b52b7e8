"""cudaHostRegister cost vs staged copies for a 218 MB pageable source."""
import time
import numpy as np
import torch

nb = 218 << 20
x = np.random.default_rng(0).integers(0, 255, nb, dtype=np.uint8)
d = torch.empty(nb, dtype=torch.uint8, device="cuda")
cr = torch.cuda.cudart()
for rep in range(3):
    t0 = time.perf_counter()
    r = cr.cudaHostRegister(x.ctypes.data, nb, 0)
    t1 = time.perf_counter()
    d.copy_(torch.from_numpy(x), non_blocking=True)
    torch.cuda.synchronize()
    t2 = time.perf_counter()
    cr.cudaHostUnregister(x.ctypes.data)
    t3 = time.perf_counter()
    print(f"register {1e3*(t1-t0):.2f} ms (rc {r}), copy {1e3*(t2-t1):.2f} ms = {nb/(t2-t1)/1e9:.1f} GB/s, "
          f"unregister {1e3*(t3-t2):.2f} ms", flush=True)
