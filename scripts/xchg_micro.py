"""Host cost of the pieces of TorchExchange.exchange at one rank (NCCL):
meta upload, counts all-to-all + readback, send wrap, rows all-to-all."""
import os, time, sys
sys.path.insert(0, ".")
import numpy as np, torch, torch.distributed as dist
from paper_2311_02206_b200.partition import CudaBuffer
os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT="29533")
torch.cuda.set_device(0)
dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
buf = torch.empty(1 << 20, dtype=torch.int64, device="cuda")
recv = torch.empty(1 << 20, dtype=torch.int64, device="cuda")
N = 500
def tm(name, f):
    for _ in range(20): f()
    torch.cuda.synchronize(); t = time.perf_counter()
    for _ in range(N): f()
    torch.cuda.synchronize(); print(f"{name:40s} {(time.perf_counter() - t) / N * 1e6:8.1f} us", flush=True)
counts = np.array([1000], dtype=np.uint64)
meta_np = lambda: np.stack([counts.astype(np.int64), np.full(1, 5, dtype=np.int64)], 1).reshape(-1)
tm("np meta build", meta_np)
tm("as_tensor(meta, cuda)", lambda: torch.as_tensor(meta_np(), device="cuda"))
pin = torch.empty(2, dtype=torch.int64).pin_memory()
def up():
    pin.numpy()[:] = meta_np(); return pin.to("cuda", non_blocking=True)
tm("pinned meta upload", up)
m = torch.as_tensor(meta_np(), device="cuda"); r = torch.empty_like(m)
tm("all_to_all_single(meta)", lambda: dist.all_to_all_single(r, m))
tm("all_to_all + .cpu()", lambda: (dist.all_to_all_single(r, m), r.cpu()))
tm("as_tensor(CudaBuffer)", lambda: torch.as_tensor(CudaBuffer(buf.data_ptr(), 1000), device="cuda"))
tm("rows all_to_all_single(splits)", lambda: dist.all_to_all_single(recv[:1000], buf[:1000], [1000], [1000]))
tm("rows all_to_all_single(nosplit)", lambda: dist.all_to_all_single(recv[:1000], buf[:1000]))
dist.destroy_process_group()
