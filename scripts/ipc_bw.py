"""P2P bandwidth through CUDA IPC mappings between two processes (the copy-
engine transport's path): rank 1 maps rank 0's 1 GiB buffer and pushes into
it with cudaMemcpyAsync (copy engine) and with the SM span-copy kernel.
torchrun --nproc-per-node 2 scripts/ipc_bw.py"""
import ctypes as C, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import torch.distributed as dist
import paper_2510_18121_b200._native as N
from paper_2510_18121_b200._native import lib, check

rank = int(os.environ["RANK"])
torch.cuda.set_device(rank)
dist.init_process_group("nccl", device_id=torch.device("cuda", rank))
NB = 1 << 30
buf = torch.zeros(NB, dtype=torch.uint8, device="cuda")
hb = (N.u8 * 64)()
off = N.i64()
check(lib().cad_ipc_handle(buf.data_ptr(), hb, C.byref(off)))
allh = [None, None]
dist.all_gather_object(allh, (bytes(hb), off.value))
if rank == 1:
    base = C.c_void_p()
    check(lib().cad_ipc_open((N.u8 * 64).from_buffer_copy(allh[0][0]), C.byref(base)))
    dst = base.value + allh[0][1]
    src = torch.empty(NB, dtype=torch.uint8, device="cuda").random_()
    s = torch.cuda.current_stream()

    def timed(fn, reps=5):
        fn(); torch.cuda.synchronize()
        t = time.perf_counter()
        for _ in range(reps):
            fn()
        torch.cuda.synchronize()
        return (time.perf_counter() - t) / reps

    runs = (N.cad_run * 1)()
    runs[0] = N.cad_run(0, 0, NB // 4096)
    t = timed(lambda: check(lib().cad_copy_runs(runs, 1, src.data_ptr(), dst, 4096, s.cuda_stream)))
    print(f"IPC copy engine, 1 memcpy of 1 GiB: {NB / t / 1e9:.1f} GB/s", flush=True)
    runs64 = (N.cad_run * 64)()
    for i in range(64):
        runs64[i] = N.cad_run(i * (NB // 4096 // 64), i * (NB // 4096 // 64), NB // 4096 // 64)
    t = timed(lambda: check(lib().cad_copy_runs(runs64, 64, src.data_ptr(), dst, 4096, s.cuda_stream)))
    print(f"IPC copy engine, 64 memcpys of 16 MiB: {NB / t / 1e9:.1f} GB/s", flush=True)
    spans = torch.tensor([[src.data_ptr(), dst, NB]], dtype=torch.int64, device="cuda")
    for n in (2, 8, 32):
        t = timed(lambda: check(lib().cad_copy_spans(spans.data_ptr(), 1, n, s.cuda_stream)))
        print(f"IPC SM copy, {n} CTAs: {NB / t / 1e9:.1f} GB/s", flush=True)
    # the transports' shape: ~40 spans of 2 MB (rows of a few tasks)
    sp = torch.tensor([[src.data_ptr() + i * (2 << 20), dst + i * (2 << 20), 2 << 20] for i in range(40)],
                      dtype=torch.int64, device="cuda")
    for n in (4, 8):
        t = timed(lambda: check(lib().cad_copy_spans(sp.data_ptr(), 40, n, s.cuda_stream)))
        print(f"IPC SM copy, 40 x 2 MiB spans, {n} CTAs: {80 * (1 << 20) / t / 1e9:.1f} GB/s", flush=True)
    runs40 = (N.cad_run * 40)()
    for i in range(40):
        runs40[i] = N.cad_run(i * 512, i * 512, 512)
    t = timed(lambda: check(lib().cad_copy_runs(runs40, 40, src.data_ptr(), dst, 4096, s.cuda_stream)))
    print(f"IPC copy engine, 40 memcpys of 2 MiB: {80 * (1 << 20) / t / 1e9:.1f} GB/s", flush=True)
    check(lib().cad_ipc_close(base.value))
dist.barrier()
dist.destroy_process_group()
