// Dispatch/return data movement: NCCL all-to-allv over NVLink (grouped
// ncclSend/ncclRecv on a caller stream) and the row gather/scatter kernels
// that pack per-peer send buffers and unpack received rows into the server
// (or home) layouts of cad_layer_plan.
//
// NCCL is bound at run time (dlopen of libnccl.so.2): inside a process that
// already runs torch.distributed this resolves to the NCCL torch loaded, so
// both communicators share one library.
#define CAD_KERNEL_TAG "comm"  // names this file in the mbarrier-timeout report
#include <cuda.h>
#include <cudaTypedefs.h>
#include <cuda_bf16.h>
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdlib>
#include <cstring>
#include <memory>
#include <mutex>
#include <string>

#include "../host/cad_status.hpp"
#include "ca_common.cuh"
#include "sm100.cuh"

namespace {

struct Nccl {
  void* h = nullptr;
  decltype(&ncclGetUniqueId) get_id = nullptr;
  decltype(&ncclCommInitRank) init_rank = nullptr;
  decltype(&ncclCommDestroy) destroy = nullptr;
  decltype(&ncclGroupStart) group_start = nullptr;
  decltype(&ncclGroupEnd) group_end = nullptr;
  decltype(&ncclSend) send = nullptr;
  decltype(&ncclRecv) recv = nullptr;
  decltype(&ncclGetErrorString) err = nullptr;
};

const Nccl& nccl() {
  static Nccl n;
  static std::string load_error;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      const char* e = dlerror();  // read once: a second call returns NULL
      load_error = e ? e : "dlopen failed";
      return;
    }
    n.h = h;
    n.get_id = reinterpret_cast<decltype(n.get_id)>(dlsym(h, "ncclGetUniqueId"));
    n.init_rank = reinterpret_cast<decltype(n.init_rank)>(dlsym(h, "ncclCommInitRank"));
    n.destroy = reinterpret_cast<decltype(n.destroy)>(dlsym(h, "ncclCommDestroy"));
    n.group_start = reinterpret_cast<decltype(n.group_start)>(dlsym(h, "ncclGroupStart"));
    n.group_end = reinterpret_cast<decltype(n.group_end)>(dlsym(h, "ncclGroupEnd"));
    n.send = reinterpret_cast<decltype(n.send)>(dlsym(h, "ncclSend"));
    n.recv = reinterpret_cast<decltype(n.recv)>(dlsym(h, "ncclRecv"));
    n.err = reinterpret_cast<decltype(n.err)>(dlsym(h, "ncclGetErrorString"));
  });
  if (!n.h) throw cad::NcclError("libnccl.so.2 unavailable: " + load_error);
  if (!n.get_id || !n.init_rank || !n.destroy || !n.group_start || !n.group_end || !n.send || !n.recv)
    throw cad::NcclError("libnccl.so.2 lacks a required symbol");
  return n;
}

void nccl_check(ncclResult_t r, const char* what) {
  if (r == ncclSuccess) return;
  const Nccl& n = nccl();
  const char* msg = n.err ? n.err(r) : nullptr;
  throw cad::NcclError(std::string(what) + ": " + (msg ? msg : ("ncclResult " + std::to_string(int(r)))));
}

// ------------------------------------------------------------------ kernels
__global__ void gather_rows_kernel(const uint4* __restrict__ src, const int64_t* __restrict__ idx,
                                   int64_t n, int64_t chunks, uint4* __restrict__ dst) {
  const int64_t total = n * chunks;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = t / chunks, c = t - r * chunks;
    dst[t] = src[idx[r] * chunks + c];
  }
}

__global__ void scatter_rows_kernel(const uint4* __restrict__ src, const int64_t* __restrict__ idx,
                                    int64_t n, int64_t chunks, uint4* __restrict__ dst) {
  const int64_t total = n * chunks;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = t / chunks, c = t - r * chunks;
    dst[idx[r] * chunks + c] = src[t];
  }
}

// 8 bf16 per thread added into 8 fp32 (atomic: a row may repeat).
__global__ void scatter_add_bf16_kernel(const uint4* __restrict__ src, const int64_t* __restrict__ idx,
                                        int64_t n, int64_t chunks, float* __restrict__ dst) {
  const int64_t total = n * chunks;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t r = t / chunks, c = t - r * chunks;
    const uint4 v = src[t];
    const __nv_bfloat162* b = reinterpret_cast<const __nv_bfloat162*>(&v);
    float* d = dst + (idx[r] * chunks + c) * 8;
#pragma unroll
    for (int i = 0; i < 4; ++i) {
      const float2 f = __bfloat1622float2(b[i]);
      atomicAdd(d + 2 * i, f.x);
      atomicAdd(d + 2 * i + 1, f.y);
    }
  }
}

__global__ void gather_cols_kernel(const float* __restrict__ src, int64_t src_rows, int heads,
                                   const int64_t* __restrict__ idx, int64_t n, float* __restrict__ dst) {
  const int64_t total = n * heads;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = t / heads, h = t - i * heads;
    dst[t] = src[h * src_rows + idx[i]];
  }
}

__global__ void scatter_cols_kernel(const float* __restrict__ src, const int64_t* __restrict__ idx, int64_t n,
                                    int heads, float* __restrict__ dst, int64_t dst_rows) {
  const int64_t total = n * heads;
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < total; t += int64_t(gridDim.x) * blockDim.x) {
    const int64_t i = t / heads, h = t - i * heads;
    dst[h * dst_rows + idx[i]] = src[t];
  }
}

__global__ void f32_to_bf16_kernel(const float4* __restrict__ src, int64_t n4, uint2* __restrict__ dst) {
  for (int64_t t = blockIdx.x * int64_t(blockDim.x) + threadIdx.x; t < n4; t += int64_t(gridDim.x) * blockDim.x) {
    const float4 f = src[t];
    __nv_bfloat162 a = __floats2bfloat162_rn(f.x, f.y), b = __floats2bfloat162_rn(f.z, f.w);
    uint2 o;
    std::memcpy(&o.x, &a, 4);
    std::memcpy(&o.y, &b, 4);
    dst[t] = o;
  }
}

unsigned blocks_for(int64_t work) {
  const int64_t b = (work + 255) / 256;
  return static_cast<unsigned>(std::max<int64_t>(1, std::min<int64_t>(b, 148 * 16)));
}

}  // namespace

namespace {

PFN_cuStreamWriteValue32_v11070 write_value_fn() {
  static PFN_cuStreamWriteValue32_v11070 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuStreamWriteValue32", &p, 11070, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuStreamWriteValue32_v11070>(p);
  });
  if (!fn) throw cad::CudaError("cuStreamWriteValue32 unavailable");
  return fn;
}

PFN_cuStreamWaitValue32_v11070 wait_value_fn() {
  static PFN_cuStreamWaitValue32_v11070 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuStreamWaitValue32", &p, 11070, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuStreamWaitValue32_v11070>(p);
  });
  if (!fn) throw cad::CudaError("cuStreamWaitValue32 unavailable");
  return fn;
}

PFN_cuMemGetAddressRange_v3020 addr_range_fn() {
  static PFN_cuMemGetAddressRange_v3020 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPointByVersion("cuMemGetAddressRange", &p, 3020, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuMemGetAddressRange_v3020>(p);
  });
  if (!fn) throw cad::CudaError("cuMemGetAddressRange unavailable");
  return fn;
}

}  // namespace

struct cad_comm {
  ncclComm_t comm = nullptr;
  int32_t rank = 0, world = 1;
};

namespace cad_dev {

// Grid-stride copy of a span list: span i is cut into 64 KB chunks, chunk c
// of the concatenation goes to CTA c % gridDim.x. 16-byte vectors when the
// span is 16-byte aligned, 4-byte words otherwise.
__global__ void __launch_bounds__(512) copy_spans_kernel(const cad_span* spans, int64_t n) {
  constexpr int64_t kChunk = 65536;
  int64_t base = 0;  // first chunk index of span i
  for (int64_t i = 0; i < n; ++i) {
    const cad_span sp = spans[i];
    const int64_t chunks = (sp.bytes + kChunk - 1) / kChunk;
    int64_t c = (blockIdx.x - base % gridDim.x + gridDim.x) % gridDim.x;  // my first chunk of this span
    for (; c < chunks; c += gridDim.x) {
      const int64_t off = c * kChunk;
      const int64_t len = min(kChunk, sp.bytes - off);
      const char* src = static_cast<const char*>(sp.src) + off;
      char* dst = static_cast<char*>(sp.dst) + off;
      if (((reinterpret_cast<uintptr_t>(src) | reinterpret_cast<uintptr_t>(dst) | len) & 15) == 0) {
        const int4* s4 = reinterpret_cast<const int4*>(src);
        int4* d4 = reinterpret_cast<int4*>(dst);
        const int64_t nv = len / 16;
        int64_t k = threadIdx.x;
        for (; k + 3 * 512 < nv; k += 4 * 512) {
          const int4 a = s4[k], b = s4[k + 512], c2 = s4[k + 1024], d = s4[k + 1536];
          d4[k] = a;
          d4[k + 512] = b;
          d4[k + 1024] = c2;
          d4[k + 1536] = d;
        }
        for (; k < nv; k += 512) d4[k] = s4[k];
      } else {
        const int* s1 = reinterpret_cast<const int*>(src);
        int* d1 = reinterpret_cast<int*>(dst);
        for (int64_t k = threadIdx.x; k < len / 4; k += 512) d1[k] = s1[k];
      }
    }
    base += chunks;
  }
}


// TMA bulk variant (one CTA per SM left free by the CA kernels): thread 0
// streams 16-byte aligned spans in batches of kBulkBufs 32 KB chunks,
// global -> shared (mbarrier complete_tx) -> global (dst may be a peer
// mapping: the write crosses NVLink). Spans that are not 16-byte aligned
// (LSE columns) are copied by all threads with 4-byte words.
constexpr int kBulkChunk = 32768, kBulkBufs = 6;
constexpr int kBulkSmem = kBulkChunk * kBulkBufs;

__global__ void __launch_bounds__(256) copy_spans_bulk_kernel(const cad_span* spans, int64_t n) {
  extern __shared__ __align__(128) uint8_t cbuf[];
  __shared__ uint64_t bar[kBulkBufs];
  if (threadIdx.x == 0) {
    for (int i = 0; i < kBulkBufs; ++i) mbar_init(&bar[i], 1);
    fence_barrier_init();
  }
  __syncthreads();
  // unaligned spans: word copies, chunks dealt round-robin over the CTAs
  int64_t base = 0;
  for (int64_t i = 0; i < n; ++i) {
    const cad_span sp = spans[i];
    const bool aligned = ((reinterpret_cast<uintptr_t>(sp.src) | reinterpret_cast<uintptr_t>(sp.dst) |
                           static_cast<uint64_t>(sp.bytes)) & 15) == 0;
    const int64_t chunks = (sp.bytes + kBulkChunk - 1) / kBulkChunk;
    if (!aligned) {
      for (int64_t c = (blockIdx.x - base % gridDim.x + gridDim.x) % gridDim.x; c < chunks; c += gridDim.x) {
        const int64_t off = c * kBulkChunk, len = min(int64_t(kBulkChunk), sp.bytes - off);
        const int* s1 = reinterpret_cast<const int*>(static_cast<const char*>(sp.src) + off);
        int* d1 = reinterpret_cast<int*>(static_cast<char*>(sp.dst) + off);
        for (int64_t k = threadIdx.x; k < len / 4; k += blockDim.x) d1[k] = s1[k];
      }
    }
    base += chunks;
  }
  if (threadIdx.x != 0) return;
  const uint32_t sb = smem_u32(cbuf);
  uint32_t phase = 0;  // all slots complete one phase per batch
  int nb = 0;          // loads in the current batch
  const char* bdst[kBulkBufs];
  int blen[kBulkBufs];
  auto flush = [&]() {
    for (int s = 0; s < nb; ++s) {
      mbar_wait(&bar[s], phase);
      asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;"
                   :: "l"(bdst[s]), "r"(sb + s * kBulkChunk), "r"(blen[s]) : "memory");
    }
    asm volatile("cp.async.bulk.commit_group;" ::: "memory");
    asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");  // slots reusable
    phase ^= 1;
    nb = 0;
  };
  base = 0;
  for (int64_t i = 0; i < n; ++i) {
    const cad_span sp = spans[i];
    const bool aligned = ((reinterpret_cast<uintptr_t>(sp.src) | reinterpret_cast<uintptr_t>(sp.dst) |
                           static_cast<uint64_t>(sp.bytes)) & 15) == 0;
    const int64_t chunks = (sp.bytes + kBulkChunk - 1) / kBulkChunk;
    if (aligned) {
      for (int64_t c = (blockIdx.x - base % gridDim.x + gridDim.x) % gridDim.x; c < chunks; c += gridDim.x) {
        const int64_t off = c * kBulkChunk;
        const int len = static_cast<int>(min(int64_t(kBulkChunk), sp.bytes - off));
        mbar_expect_tx(&bar[nb], len);
        asm volatile(
            "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
            :: "r"(sb + nb * kBulkChunk), "l"(static_cast<const char*>(sp.src) + off), "r"(len),
               "r"(smem_u32(&bar[nb])) : "memory");
        bdst[nb] = static_cast<const char*>(sp.dst) + off;
        blen[nb] = len;
        if (++nb == kBulkBufs) flush();
      }
    }
    base += chunks;
  }
  if (nb) flush();
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");  // stores complete before exit
}
void preload_comm() {
  cudaFuncAttributes a;
  for (const void* f : {reinterpret_cast<const void*>(gather_rows_kernel), reinterpret_cast<const void*>(scatter_rows_kernel),
                        reinterpret_cast<const void*>(scatter_add_bf16_kernel),
                        reinterpret_cast<const void*>(gather_cols_kernel),
                        reinterpret_cast<const void*>(scatter_cols_kernel),
                        reinterpret_cast<const void*>(f32_to_bf16_kernel), reinterpret_cast<const void*>(copy_spans_kernel)})
    cuda_check(cudaFuncGetAttributes(&a, f), "load comm kernels");
  set_max_smem(reinterpret_cast<const void*>(copy_spans_bulk_kernel), kBulkSmem, "cudaFuncSetAttribute(copy_spans_bulk)");
}
}  // namespace cad_dev

extern "C" {

int cad_comm_unique_id(uint8_t id[CAD_UNIQUE_ID_BYTES]) {
  return cad::guarded([&] {
    static_assert(sizeof(ncclUniqueId) == CAD_UNIQUE_ID_BYTES, "unique id size");
    ncclUniqueId u;
    nccl_check(nccl().get_id(&u), "ncclGetUniqueId");
    std::memcpy(id, &u, sizeof(u));
  });
}

int cad_comm_init(const uint8_t id[CAD_UNIQUE_ID_BYTES], int32_t rank, int32_t world, cad_comm** comm) {
  return cad::guarded([&] {
    if (!id || !comm || world < 1 || rank < 0 || rank >= world) throw cad::DomainError("bad argument");
    ncclUniqueId u;
    std::memcpy(&u, id, sizeof(u));
    auto c = std::make_unique<cad_comm>();
    c->rank = rank;
    c->world = world;
    nccl_check(nccl().init_rank(&c->comm, world, u, rank), "ncclCommInitRank");
    *comm = c.release();
  });
}

int cad_comm_destroy(cad_comm* comm) {
  return cad::guarded([&] {
    if (!comm) return;
    if (comm->comm) nccl_check(nccl().destroy(comm->comm), "ncclCommDestroy");
    delete comm;
  });
}

int cad_alltoallv(cad_comm* comm, const void* send, const int64_t* send_bytes, const int64_t* send_displ,
                  void* recv, const int64_t* recv_bytes, const int64_t* recv_displ, void* stream) {
  return cad::guarded([&] {
    if (!comm || !send_bytes || !send_displ || !recv_bytes || !recv_displ) throw cad::DomainError("null argument");
    const Nccl& n = nccl();
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    nccl_check(n.group_start(), "ncclGroupStart");
    for (int32_t p = 0; p < comm->world; ++p) {
      if (send_bytes[p] > 0)
        nccl_check(n.send(static_cast<const char*>(send) + send_displ[p], static_cast<size_t>(send_bytes[p]), ncclUint8,
                          p, comm->comm, s),
                   "ncclSend");
      if (recv_bytes[p] > 0)
        nccl_check(n.recv(static_cast<char*>(recv) + recv_displ[p], static_cast<size_t>(recv_bytes[p]), ncclUint8, p,
                          comm->comm, s),
                   "ncclRecv");
    }
    nccl_check(n.group_end(), "ncclGroupEnd");
  });
}

int cad_gather_rows(const void* src, const int64_t* idx, int64_t n, int64_t row_bytes, void* dst, void* stream) {
  return cad::guarded([&] {
    if (n == 0) return;
    if (!src || !idx || !dst || row_bytes % 16) throw cad::DomainError("bad gather arguments");
    const int64_t chunks = row_bytes / 16;
    gather_rows_kernel<<<blocks_for(n * chunks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(src), idx, n, chunks, static_cast<uint4*>(dst));
    cad_dev::cuda_check(cudaGetLastError(), "gather_rows");
  });
}

int cad_scatter_rows(const void* src, const int64_t* idx, int64_t n, int64_t row_bytes, void* dst, void* stream) {
  return cad::guarded([&] {
    if (n == 0) return;
    if (!src || !idx || !dst || row_bytes % 16) throw cad::DomainError("bad scatter arguments");
    const int64_t chunks = row_bytes / 16;
    scatter_rows_kernel<<<blocks_for(n * chunks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(src), idx, n, chunks, static_cast<uint4*>(dst));
    cad_dev::cuda_check(cudaGetLastError(), "scatter_rows");
  });
}

int cad_scatter_add_bf16(const void* src, const int64_t* idx, int64_t n, int64_t row_elems, float* dst,
                         void* stream) {
  return cad::guarded([&] {
    if (n == 0) return;
    if (!src || !idx || !dst || row_elems % 8) throw cad::DomainError("bad scatter-add arguments");
    const int64_t chunks = row_elems / 8;
    scatter_add_bf16_kernel<<<blocks_for(n * chunks), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        static_cast<const uint4*>(src), idx, n, chunks, dst);
    cad_dev::cuda_check(cudaGetLastError(), "scatter_add_bf16");
  });
}

int cad_gather_cols_f32(const float* src, int64_t src_rows, int32_t heads, const int64_t* idx, int64_t n, float* dst,
                        void* stream) {
  return cad::guarded([&] {
    if (n == 0) return;
    if (!src || !idx || !dst) throw cad::DomainError("null argument");
    gather_cols_kernel<<<blocks_for(n * heads), 256, 0, static_cast<cudaStream_t>(stream)>>>(src, src_rows, heads,
                                                                                               idx, n, dst);
    cad_dev::cuda_check(cudaGetLastError(), "gather_cols");
  });
}

int cad_scatter_cols_f32(const float* src, const int64_t* idx, int64_t n, int32_t heads, float* dst,
                         int64_t dst_rows, void* stream) {
  return cad::guarded([&] {
    if (n == 0) return;
    if (!src || !idx || !dst) throw cad::DomainError("null argument");
    scatter_cols_kernel<<<blocks_for(n * heads), 256, 0, static_cast<cudaStream_t>(stream)>>>(src, idx, n, heads,
                                                                                                dst, dst_rows);
    cad_dev::cuda_check(cudaGetLastError(), "scatter_cols");
  });
}

int cad_f32_to_bf16(const float* src, int64_t n, void* dst, void* stream) {
  return cad::guarded([&] {
    if (n == 0) return;
    if (!src || !dst || n % 4) throw cad::DomainError("bad conversion arguments");
    f32_to_bf16_kernel<<<blocks_for(n / 4), 256, 0, static_cast<cudaStream_t>(stream)>>>(
        reinterpret_cast<const float4*>(src), n / 4, static_cast<uint2*>(dst));
    cad_dev::cuda_check(cudaGetLastError(), "f32_to_bf16");
  });
}

int cad_ipc_handle(const void* ptr, uint8_t handle[64], int64_t* offset) {
  return cad::guarded([&] {
    if (!ptr || !handle || !offset) throw cad::DomainError("null argument");
    CUdeviceptr base = 0;
    size_t size = 0;
    if (addr_range_fn()(&base, &size, reinterpret_cast<CUdeviceptr>(ptr)) != CUDA_SUCCESS)
      throw cad::CudaError("cuMemGetAddressRange failed");
    cudaIpcMemHandle_t h;
    cad_dev::cuda_check(cudaIpcGetMemHandle(&h, reinterpret_cast<void*>(base)), "cudaIpcGetMemHandle");
    static_assert(sizeof(h) == 64, "ipc handle size");
    std::memcpy(handle, &h, 64);
    *offset = static_cast<int64_t>(reinterpret_cast<CUdeviceptr>(ptr) - base);
  });
}

int cad_ipc_open(const uint8_t handle[64], void** base) {
  return cad::guarded([&] {
    if (!handle || !base) throw cad::DomainError("null argument");
    cudaIpcMemHandle_t h;
    std::memcpy(&h, handle, 64);
    cad_dev::cuda_check(cudaIpcOpenMemHandle(base, h, cudaIpcMemLazyEnablePeerAccess), "cudaIpcOpenMemHandle");
  });
}

int cad_ipc_close(void* base) {
  return cad::guarded([&] {
    if (base) cad_dev::cuda_check(cudaIpcCloseMemHandle(base), "cudaIpcCloseMemHandle");
  });
}

int cad_copy_runs(const cad_run* runs, int64_t n, const void* src, void* dst, int64_t row_bytes, void* stream) {
  return cad::guarded([&] {
    if (n == 0) return;
    if (!runs || !src || !dst) throw cad::DomainError("null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int64_t i = 0; i < n; ++i) {
      const cad_run& r = runs[i];
      cad_dev::cuda_check(cudaMemcpyAsync(static_cast<char*>(dst) + r.dst_row * row_bytes,
                                          static_cast<const char*>(src) + r.src_row * row_bytes,
                                          static_cast<size_t>(r.n_rows * row_bytes), cudaMemcpyDeviceToDevice, s),
                          "cudaMemcpyAsync(run)");
    }
  });
}

int cad_copy_spans(const cad_span* spans, int64_t n, int32_t n_ctas, void* stream) {
  return cad::guarded([&] {
    if (n == 0) return;
    if (!spans || n_ctas < 1) throw cad::DomainError("bad argument");
    static const bool simt = std::getenv("CAD_COPY_SIMT") != nullptr;
    if (simt) {
      cad_dev::copy_spans_kernel<<<n_ctas, 512, 0, static_cast<cudaStream_t>(stream)>>>(spans, n);
    } else {
      cad_dev::set_max_smem(reinterpret_cast<const void*>(cad_dev::copy_spans_bulk_kernel), cad_dev::kBulkSmem,
                            "cudaFuncSetAttribute(copy_spans_bulk)");
      cad_dev::copy_spans_bulk_kernel<<<n_ctas, 256, cad_dev::kBulkSmem, static_cast<cudaStream_t>(stream)>>>(
          spans, n);
    }
    cad_dev::cuda_check(cudaGetLastError(), "copy_spans launch");
  });
}

int cad_copy_runs_cols(const cad_run* runs, int64_t n, const float* src, int64_t src_rows, float* dst,
                       int64_t dst_rows, int32_t heads, void* stream) {
  return cad::guarded([&] {
    if (n == 0) return;
    if (!runs || !src || !dst) throw cad::DomainError("null argument");
    cudaStream_t s = static_cast<cudaStream_t>(stream);
    for (int64_t i = 0; i < n; ++i) {
      const cad_run& r = runs[i];
      cad_dev::cuda_check(cudaMemcpy2DAsync(dst + r.dst_row, static_cast<size_t>(dst_rows) * 4, src + r.src_row,
                                            static_cast<size_t>(src_rows) * 4, static_cast<size_t>(r.n_rows) * 4,
                                            static_cast<size_t>(heads), cudaMemcpyDeviceToDevice, s),
                          "cudaMemcpy2DAsync(run)");
    }
  });
}

int cad_stream_write_u32(void* addr, uint32_t value, void* stream) {
  return cad::guarded([&] {
    if (!addr) throw cad::DomainError("null argument");
    if (write_value_fn()(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value,
                         CU_STREAM_WRITE_VALUE_DEFAULT) != CUDA_SUCCESS)
      throw cad::CudaError("cuStreamWriteValue32 failed");
  });
}

int cad_stream_wait_u32(const void* addr, uint32_t value, void* stream) {
  return cad::guarded([&] {
    if (!addr) throw cad::DomainError("null argument");
    if (wait_value_fn()(static_cast<CUstream>(stream), reinterpret_cast<CUdeviceptr>(addr), value,
                        CU_STREAM_WAIT_VALUE_GEQ) != CUDA_SUCCESS)
      throw cad::CudaError("cuStreamWaitValue32 failed");
  });
}

}  // extern "C"
