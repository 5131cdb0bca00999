"""Build lib/libcad_tl_dkdv.so: the dK/dV kernel with clock64 trace points in
block 0 (per iteration i of the unit loop); read by scripts/timeline_dkdv.py.
Debug tool only."""
import os, re, subprocess
PKG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2510_18121_b200")
s = open(os.path.join(PKG, "csrc/cuda/ca_bwd.cu")).read()
s = """#include <cstdint>
__device__ unsigned long long g_tl[24][8192];
#define TL(ev, it) do { if (blockIdx.x == 0 && (it) < 8192) { uint64_t t_; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_)); g_tl[ev][it] = t_; } } while (0)
""" + s
a, b = s.index("ca_bwd_dkdv_kernel("), s.index("}  // namespace kv")
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
rep(r"mbar_wait\(&bars->p_full, p_ph\);", L + "TL(7, tli + i);", L + "TL(0, tli + i);")
rep(r"mma_commit\(&bars->s_full\);", post=L + "TL(8, tli + i);", nth=1)
rep(r"mbar_wait\(&bars->ds_full, ds_ph\);", L + "TL(13, tli + i);", L + "TL(1, tli + i);")
rep(r"mma_commit\(&bars->q_empty\[qcur\]\);.*", post=L + "TL(9, tli + i);")
rep(r"mma_commit\(&bars->dp_full\);", post=L + "TL(10, tli + i);", nth=1)
rep(r"mbar_wait\(&bars->q_full\[qr\.i\], qr\.ph\);", L + "TL(11, tli + i);", L + "TL(12, tli + i);", nth=1)
W1 = "else if (threadIdx.x == 128) "
rep(r"mbar_wait_warp\(&bars->s_full, s_ph\);", W + "TL(2, tli + i); " + W1 + "TL(14, tli + i);", W + "TL(3, tli + i); " + W1 + "TL(15, tli + i);")
rep(r"mbar_arrive\(ch \? &bars->p_full : &bars->p_half\);", post="if (ch) { " + W + "TL(4, tli + i); " + W1 + "TL(16, tli + i); }")
rep(r"mbar_wait_warp\(&bars->dp_full, dp_ph\);", post=W + "TL(5, tli + i); " + W1 + "TL(17, tli + i);")
rep(r"mbar_arrive\(ch \? &bars->ds_full : &bars->ds_half\);", post="if (ch) { " + W + "TL(6, tli + i); " + W1 + "TL(18, tli + i); }")
# trace index = position of the iteration in this CTA's work list
decl = "const KvUnit un = p.units[u];"
parts = k.split(decl)
assert len(parts) == 4, len(parts)  # producer, MMA, elementwise
k = parts[0] + decl + parts[1] + decl + " tli = tl_next; tl_next += un.n_iter;" + parts[2] + decl + \
    " tli = tl_next; tl_next += un.n_iter;" + parts[3]
k = k.replace("    } else if (warp == 9) {", "    } else if (warp == 9) {\n      int tli = 0, tl_next = 0;", 1)
k = k.replace('    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");',
              '    asm volatile("setmaxnreg.inc.sync.aligned.u32 208;");\n    int tli = 0, tl_next = 0;', 1)
s = s[:a] + k + s[b:]
s += """
extern "C" int cad_debug_timeline(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_tl, sizeof(g_tl)) == cudaSuccess ? 0 : -3;
}
"""
tmp = os.path.join(PKG, "csrc/cuda/_tl_bwd.cu")
open(tmp, "w").write(s)
try:
    subprocess.run(["nvcc", "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
                    "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-c", tmp, "-o", "/tmp/_tl_bwd.o"], check=True)
finally:
    os.remove(tmp)
bd = os.path.join(PKG, "build")
objs = [os.path.join(bd, f) for f in sorted(os.listdir(bd)) if f.endswith(".o") and f != "cuda_ca_bwd.o"]
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                os.path.join(PKG, "lib/libcad_tl_dkdv.so"), *objs, "/tmp/_tl_bwd.o", "-ldl", "-lpthread"], check=True)
