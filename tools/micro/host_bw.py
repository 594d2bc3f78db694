import numpy as np, time, os, torch
n = 890_000_000
src = np.random.randint(0, 200, n, dtype=np.uint8)
dst = torch.empty(n, dtype=torch.int32, pin_memory=True).numpy().view(np.uint32)
dst2 = np.empty(n, np.uint32)
for name, d in (("pinned", dst), ("pageable", dst2)):
    t = time.perf_counter(); np.copyto(d, src, casting="unsafe"); t1 = time.perf_counter()
    np.copyto(d, src, casting="unsafe"); t2 = time.perf_counter()
    print(name, "widen 1 thread", f"{1e3*(t2-t1):.1f} ms", f"{n*5/(t2-t1)/1e9:.1f} GB/s")
print("cpus", os.cpu_count(), len(os.sched_getaffinity(0)))
a = torch.empty(n, dtype=torch.int32, pin_memory=True); g = torch.empty(n, dtype=torch.int32, device="cuda")
torch.cuda.synchronize()
for i in range(2):
    t=time.perf_counter(); a.copy_(g); torch.cuda.synchronize(); t1=time.perf_counter()
print("D2H 3.56 GB", f"{1e3*(t1-t):.1f} ms", f"{n*4/(t1-t)/1e9:.1f} GB/s")
b = torch.empty(n, dtype=torch.uint8, pin_memory=True); g8 = torch.empty(n, dtype=torch.uint8, device="cuda")
for i in range(2):
    t=time.perf_counter(); b.copy_(g8); torch.cuda.synchronize(); t1=time.perf_counter()
print("D2H 0.89 GB", f"{1e3*(t1-t):.1f} ms", f"{n/(t1-t)/1e9:.1f} GB/s")
