"""Build lib/libcad_tl_dq.so: the dQ kernel with clock64 trace points in
block 0 (per iteration i of the unit loop); read by scripts/timeline_dq.py.
Debug tool only."""
import os, re, subprocess
PKG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2510_18121_b200")
s = open(os.path.join(PKG, "csrc/cuda/ca_bwd.cu")).read()
s = """#include <cstdint>
__device__ unsigned long long g_tl[32][8192];
#define TLV(ev, it, v) do { if (blockIdx.x == 0 && (it) < 8192) g_tl[ev][it] = (v); } while (0)
#define TL(ev, it) do { if (blockIdx.x == 0 && (it) < 8192) { uint64_t t_; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_)); g_tl[ev][it] = t_; } } while (0)
""" + s
a, b = s.index("ca_bwd_dq_kernel("), s.index("}  // namespace dq")
k = s[a:b]


def rep(pat, pre=None, post=None, nth=0):
    global k
    ms = list(re.finditer(r"^( *)(" + pat + r")$", k, re.M))
    assert ms, pat
    m = ms[nth]
    i = m.group(1)
    out = (i + pre + "\n" if pre else "") + i + m.group(2) + ("\n" + i + post if post else "")
    k = k[:m.start()] + out + k[m.end():]


L = "if (lane == 0) "
W = "if (threadIdx.x == 0) "
W1 = "else if (threadIdx.x == 128) "
# MMA warp (j loop)
rep(r"mbar_wait\(&bars->p_read, pr_ph\);", L + "{ TL(7, tli + j); TLV(24, tli + j, mbar_try(smem_u32(&bars->p_read), pr_ph)); }", L + "TL(0, tli + j);")
rep(r"mbar_wait\(&bars->kv_full\[nst\], nph\);", L + "{ TL(11, tli + j); TLV(25, tli + j, mbar_try(smem_u32(&bars->kv_full[nst]), nph)); }", L + "TL(12, tli + j);")
rep(r"mma_commit\(&bars->s_full\);", post=L + "TL(8, tli + j);", nth=1)
rep(r"mbar_wait\(&bars->ds_full, ds_ph\);", L + "{ TL(13, tli + j); TLV(26, tli + j, mbar_try(smem_u32(&bars->ds_full), ds_ph)); }", L + "TL(1, tli + j);")
rep(r"mma_commit\(&bars->kv_empty\[cur\]\);", post=L + "TL(9, tli + j);")
rep(r"mma_commit\(&bars->dp_full\);", post=L + "TL(10, tli + j);", nth=1)
# elementwise
rep(r"mbar_wait_warp\(&bars->s_full, s_ph\);", W + "TL(2, tli + j); " + W1 + "TL(14, tli + j);", W + "TL(3, tli + j); " + W1 + "TL(15, tli + j);")
rep(r"mbar_wait_warp\(&bars->dp_full, dp_ph\);", W + "TL(4, tli + j); " + W1 + "TL(16, tli + j);", W + "TL(5, tli + j); " + W1 + "TL(17, tli + j);")
rep(r"mbar_arrive\(&bars->ds_full\);", post=W + "TL(6, tli + j); " + W1 + "TL(18, tli + j);")
rep(r"mbar_arrive\(&bars->p_read\);", W + "TL(19, tli + j);", W + "TL(20, tli + j);")
rep(r"load_row64\(tDP \+ lsel \+ c0, y\);", post=W + "TL(21, tli + j);")
rep(r"tmem_wait_st\(\);", W + "TL(22, tli + j);", W + "TL(23, tli + j);")
loop = "for (int u = blockIdx.x; u < p.n_units; u += gridDim.x) {"
parts = k.split(loop)
assert len(parts) == 4, len(parts)
k = parts[0] + loop + parts[1] + "int tli = 0;\n" + loop.replace("u += ", "tli += p.units[u].n_kv, u += ") + parts[2] + \
    "int tli = 0;\n" + loop.replace("u += ", "tli += p.units[u].n_kv, u += ") + parts[3]
s = s[:a] + k + s[b:]
s += """
extern "C" int cad_debug_timeline(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_tl, sizeof(g_tl)) == cudaSuccess ? 0 : -3;
}
"""
tmp = os.path.join(PKG, "csrc/cuda/_tl_dq.cu")
open(tmp, "w").write(s)
try:
    subprocess.run(["nvcc", "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
                    "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-c", tmp, "-o", "/tmp/_tl_dq.o"], check=True)
finally:
    os.remove(tmp)
bd = os.path.join(PKG, "build")
objs = [os.path.join(bd, f) for f in sorted(os.listdir(bd)) if f.endswith(".o") and f != "cuda_ca_bwd.o"]
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                os.path.join(PKG, "lib/libcad_tl_dq.so"), *objs, "/tmp/_tl_dq.o", "-ldl", "-lpthread"], check=True)
