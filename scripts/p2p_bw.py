"""NVLink P2P bandwidth of the transports' copy methods on this box (2 GPUs, one
process): copy-engine memcpy (torch peer copy) and the SM span-copy kernels
(cad_copy_spans, SIMT and TMA bulk) with n CTAs, GPU0 -> GPU1."""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_2510_18121_b200._native import lib, check

rt = C.CDLL("libcudart.so.12") if os.path.exists("/usr/local/cuda/lib64/libcudart.so.12") else None
torch.cuda.set_device(0)
if rt is not None:
    print("enable peer 0->1:", rt.cudaDeviceEnablePeerAccess(1, 0))
N = 1 << 30
src = torch.empty(N, dtype=torch.uint8, device="cuda:0").random_()
dst = torch.empty(N, dtype=torch.uint8, device="cuda:1")
s0 = torch.cuda.current_stream(0)


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    t = time.perf_counter()
    for _ in range(reps):
        fn()
    torch.cuda.synchronize(0); torch.cuda.synchronize(1)
    return (time.perf_counter() - t) / reps


t = timed(lambda: dst.copy_(src, non_blocking=True))
print(f"copy engine (torch peer copy): {N / t / 1e9:.1f} GB/s")
spans = torch.tensor([[src.data_ptr(), dst.data_ptr(), N]], dtype=torch.int64, device="cuda:0")
for mode in ("bulk", "simt"):
    if mode == "simt":
        os.environ["CAD_COPY_SIMT"] = "1"
    for n in (2, 8, 32, 148):
        if mode == "simt" and n == 2:
            pass
        t = timed(lambda: check(lib().cad_copy_spans(spans.data_ptr(), 1, n, s0.cuda_stream)))
        print(f"SM copy ({mode}, {n} CTAs): {N / t / 1e9:.1f} GB/s")
    break  # the SIMT switch is read once per process
ok = torch.equal(dst[:1 << 20].cpu(), src[:1 << 20].cpu())
print("data ok:", ok)
