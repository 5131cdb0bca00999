"""Build lib/libcad_tl.so: a forward kernel with clock64 trace points in
block 0 (head slot 0 unless noted); read by scripts/timeline_fwd.py.
Usage: build_tl_fwd.py [single|pair]. Debug tool only."""
import os, re, subprocess, sys
PKG = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "paper_2510_18121_b200")
which = sys.argv[1] if len(sys.argv) > 1 else "single"
fname = "ca_fwd.cu" if which == "single" else "ca_fwd2.cu"
s = open(os.path.join(PKG, "csrc/cuda", fname)).read()
s = """#include <cstdint>
__device__ unsigned long long g_tlf[24][4096];
#define TL(ev, it) do { if (blockIdx.x == 0 && (it) < 4096) { uint64_t t_; asm volatile("mov.u64 %0, %%clock64;" : "=l"(t_)); g_tlf[ev][it] = t_; } } while (0)
#define SOFTMAX_TL(ev, it) if (threadIdx.x == 0) TL(ev, it)
""" + s


def rep(pat, fn, last=False):
    """Replace the first (last) line matching regex pat (whole line, any indent) by fn(indent, line)."""
    global s
    ms = list(re.finditer(r"^( *)(" + pat + r")$", s, re.M))
    assert ms, pat
    m = ms[-1] if last else ms[0]
    s = s[:m.start()] + fn(m.group(1), m.group(2)) + s[m.end():]


W = lambda ind, line, pre="", post="": (ind + pre + "\n" if pre else "") + ind + line + ("\n" + ind + post if post else "")
rep(r"mbar_wait\(&bars->p_half\[h\], pph\[h\]\);", lambda i, l: W(i, l, "if (lane == 0) TL(13 + h, tl_it + j);", "if (lane == 0) TL(8 + 3 * h, tl_it + j);"))
rep(r"mbar_wait\(&bars->p_full\[h\], pph\[h\]\);", lambda i, l: W(i, l, "if (lane == 0 && h == 0) TL(9, tl_it + j);", "if (lane == 0) TL(h ? 12 : 0, tl_it + j);"))
rep(r"(mma_commit|commit_pair)\(&bars->s_full\[h\]\);\n *\}", lambda i, l: W(i, l.replace("}", "  if (lane == 0) TL(h ? 19 : 10, tl_it + j);\n" + i[:-2] + "}")), last=True)
rep(r"mbar_wait\(&bars->v_full\[vs\], vph\);", lambda i, l: W(i, l, "if (lane == 0) TL(15, tl_it + j);", "if (lane == 0) TL(16, tl_it + j);"))
s2 = s
# the k_full wait inside the j loop (the second one in the MMA role)
idx = [m.start() for m in re.finditer(r"mbar_wait\(&bars->k_full\[ks\], kph\);", s)]
pos = idx[-1]
line_start = s.rfind("\n", 0, pos) + 1
ind = s[line_start:pos]
s = s[:line_start] + ind + "if (lane == 0) TL(17, tl_it + j);\n" + s[line_start:pos] + "mbar_wait(&bars->k_full[ks], kph);\n" + ind + "if (lane == 0) TL(18, tl_it + j);" + s[pos + len("mbar_wait(&bars->k_full[ks], kph);"):]
rep(r"mbar_wait_warp\(&bars->s_full\[h\], sph\);", lambda i, l: W(i, l, "if (row == 0 && h == 0) TL(2, tl_it + j);", "if (row == 0 && h == 0) TL(3, tl_it + j);"))
rep(r"\[&\]\(int half\) \{ (mbar_arrive|mbar_arrive_leader)\(half \? &bars->p_full\[h\] : &bars->p_half\[h\]\); \}\);",
    lambda i, l: i + l[:-2] + ", tl_it + j);\n" + i + "if (row == 0 && h == 0) TL(4, tl_it + j);")
loop = r"for \(int u = (blockIdx\.x|pair); u < p\.n_units; u \+= (gridDim\.x|n_pairs)\) \{"
for role in ("pph", "sph"):
    m = [m for m in re.finditer(loop, s) if role in s[max(0, m.start() - 200):m.start()]][0]
    st = m.group(0).replace("u += ", "tl_it += p.units[u].n_kv, u += ")
    s = s[:m.start()] + "int tl_it = 0;\n    " + st + s[m.end():]
s += """
extern "C" int cad_debug_timeline_fwd(unsigned long long* out) {
  return cudaMemcpyFromSymbol(out, g_tlf, sizeof(g_tlf)) == cudaSuccess ? 0 : -3;
}
"""
tmp = os.path.join(PKG, "csrc/cuda/_tl_fwd.cu")
open(tmp, "w").write(s)
try:
    subprocess.run(["nvcc", "-std=c++17", "-O3", "-lineinfo", "-gencode", "arch=compute_100a,code=sm_100a",
                    "--expt-relaxed-constexpr", "-Xcompiler", "-fPIC", "-c", tmp, "-o", "/tmp/_tl_fwd.o"], check=True)
finally:
    os.remove(tmp)
b = os.path.join(PKG, "build")
objs = [os.path.join(b, f) for f in sorted(os.listdir(b)) if f.endswith(".o") and f != "cuda_" + fname[:-3] + ".o"]
subprocess.run(["nvcc", "-gencode", "arch=compute_100a,code=sm_100a", "-shared", "-o",
                os.path.join(PKG, f"lib/libcad_tl_{which}.so"), *objs, "/tmp/_tl_fwd.o", "-ldl", "-lpthread"], check=True)
