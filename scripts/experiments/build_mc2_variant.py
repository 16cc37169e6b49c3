# Experiment build (not product): copies csrc/ to /tmp, patches it, builds paper_1108_0486_b200/lib/alt/libxg_gpu_<name>.so.
# usage: python <this> NAME [MACRO=VALUE ...]; A/B with scripts/gpu_lib_ab.sh or scripts/gpu_mc_ab.sh
import os, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); PKG = ROOT + "/paper_1108_0486_b200"
name, defs = sys.argv[1], sys.argv[2:]
d = f"/tmp/xg_variant_{name}"; shutil.rmtree(d, ignore_errors=True); shutil.copytree(PKG + "/csrc", d)
shutil.copy(os.path.join(os.path.dirname(os.path.abspath(__file__)), "xg_mc2_two_streams.cuh"), d + "/xg_mc2.cuh")
s = open(d + "/xg_gpu.cu").read()
s = s.replace('#include "xg_pairs.cuh"\n', '#include "xg_pairs.cuh"\n#include "xg_mc2.cuh"\n', 1)
old = "template <int MODE, class P>\nint launch_pair("
add = r'''template <class P>
int launch_mc2(const P& p, xg_ensemble* h, uint32_t g_begin, uint32_t g_count, uint64_t words,
               unsigned long long* hits, cudaStream_t s) {
    const uint64_t sms = static_cast<uint64_t>(std::max(1, h->sms));
    const uint32_t warps = g_count / 2;
    uint32_t wpb = warps > 32 * sms ? XG_MC2_WPB : static_cast<uint32_t>((warps + sms - 1) / sms);
    const unsigned grid = (warps + wpb - 1) / wpb;
    pair_kernel_mc2<P><<<grid, 32 * wpb, 0, s>>>(p, h->d_win, h->d_weyl, g_begin, g_count, words, hits);
    g_launches.fetch_add(1, std::memory_order_relaxed);
    return cuda_rc(cudaGetLastError());
}

'''
assert old in s
s = s.replace(old, add + old, 1)
old2 = "    pair_kernel<P, MODE><<<grid, 32 * wpb, smem, s>>>("
assert old2 in s
s = s.replace(old2, "    if constexpr (MODE == kMC && std::is_same_v<P, GP32>) {\n        if ((g_count & 1u) == 0 && (words & 127u) == 0) return launch_mc2(p, h, g_begin, g_count, words, hits, s);\n    }\n" + old2, 1)
open(d + "/xg_gpu.cu", "w").write(s)
out = f"{PKG}/lib/alt/libxg_gpu_{name}.so"
cmd = ["/usr/local/cuda/bin/nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
       "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-Xptxas", "-v", "-I", ROOT + "/include", *[f"-D{x}" for x in defs],
       "-o", out, d + "/xg_gpu.cu"]
r = subprocess.run(cmd, capture_output=True, text=True)
import re
for line in (r.stdout + r.stderr).splitlines():
    if "mc2" in line or "error" in line.lower(): print(line)
m = re.findall(r"Compiling entry function '(\w*mc2\w*)'.*?\n.*?Used (\d+) registers", r.stdout + r.stderr, re.S)
print(m); sys.exit(r.returncode)
