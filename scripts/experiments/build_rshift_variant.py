# Experiment build (not product): copies csrc/ to /tmp, patches it, builds paper_1108_0486_b200/lib/alt/libxg_gpu_<name>.so.
# usage: python <this> NAME [MACRO=VALUE ...]; A/B with scripts/gpu_lib_ab.sh or scripts/gpu_mc_ab.sh
# build experiment variants of libxg_gpu.so: right shifts via mul.wide.u32 (FMA pipe)
import os, re, shutil, subprocess, sys
ROOT = os.path.dirname(os.path.dirname(os.path.dirname(os.path.abspath(__file__)))); PKG = ROOT + "/paper_1108_0486_b200"
name, defs = sys.argv[1], sys.argv[2:]
d = f"/tmp/xg_variant_{name}"; shutil.rmtree(d, ignore_errors=True); shutil.copytree(PKG + "/csrc", d)
src = open(d + "/xg_pairs.cuh").read()
helper = r'''
__constant__ uint32_t c_pow2[33] = {1u,2u,4u,8u,16u,32u,64u,128u,256u,512u,1024u,2048u,4096u,8192u,16384u,32768u,65536u,
 131072u,262144u,524288u,1048576u,2097152u,4194304u,8388608u,16777216u,33554432u,67108864u,134217728u,268435456u,536870912u,1073741824u,2147483648u,0u};
// x >> r as the high word of x * 2^(32-r), multiplier opaque to ptxas
__device__ __forceinline__ uint32_t shr_wide(uint32_t x, uint32_t m) {
    uint32_t lo, hi;
    asm("{\n\t.reg .u64 t;\n\tmul.wide.u32 t, %2, %3;\n\tmov.b64 {%0, %1}, t;\n\t}" : "=r"(lo), "=r"(hi) : "r"(x), "r"(m));
    return hi;
}
__device__ __forceinline__ uint32_t xs(uint32_t x, unsigned l, unsigned r) {'''
src = src.replace("__device__ __forceinline__ uint32_t xs(uint32_t x, unsigned l, unsigned r) {", helper, 1)
# multipliers loaded once per thread (blockIdx.y == 0 always; opaque to the compiler)
src = src.replace("    uint32_t is31, not31;  // 1 / 0 on lane 31 (the GP32 giver of A.y), 0 / 1 elsewhere",
                  "    uint32_t is31, not31;  // 1 / 0 on lane 31 (the GP32 giver of A.y), 0 / 1 elsewhere\n    uint32_t mb, md, mg;")
src = src.replace("    pl.not31 = 1u - pl.is31;\n",
                  "    pl.not31 = 1u - pl.is31;\n    pl.mb = c_pow2[18 + blockIdx.y]; pl.md = c_pow2[15 + blockIdx.y]; pl.mg = c_pow2[16 + blockIdx.y];\n")
# recurrence: optionally the t>>b / t>>d shifts through shr_wide (GP32 only)
old = "    n.x = xs(A.x, p.a, p.b) ^ xs(ty, p.c, p.d);\n    n.y = xs(A.y, p.a, p.b) ^ xs(tx, p.c, p.d);\n"
assert old in src
new = r'''#if defined(XGV_D) || defined(XGV_B)
    if constexpr (std::is_same_v<P, GP32>) {
        const uint32_t t1x = A.x ^ (A.x << p.a), t2x = ty ^ (ty << p.c);
        const uint32_t t1y = A.y ^ (A.y << p.a), t2y = tx ^ (tx << p.c);
#ifdef XGV_B
        const uint32_t u1x = shr_wide(t1x, pl.mb), u1y = shr_wide(t1y, pl.mb);
#else
        const uint32_t u1x = t1x >> p.b, u1y = t1y >> p.b;
#endif
#ifdef XGV_D
        const uint32_t u2x = shr_wide(t2x, pl.md), u2y = shr_wide(t2y, pl.md);
#else
        const uint32_t u2x = t2x >> p.d, u2y = t2y >> p.d;
#endif
        n.x = t1x ^ u1x ^ t2x ^ u2x;
        n.y = t1y ^ u1y ^ t2y ^ u2y;
        return n;
    }
#endif
''' + old
src = src.replace(old, new)
# Weyl: optionally w >> gamma through shr_wide
old = "    return (w ^ (w >> p.gamma)) + v;  // xorgens.hpp:58-62\n"
assert old in src
src = src.replace("__device__ __forceinline__ uint32_t weyl_mix(uint32_t w, uint32_t v, const P& p) {\n" + old,
  "__device__ __forceinline__ uint32_t weyl_mix(uint32_t w, uint32_t v, const P& p, uint32_t mg = 0) {\n"
  "#ifdef XGV_W\n    if constexpr (std::is_same_v<P, GP32>) return (w ^ shr_wide(w, mg)) + v;\n#endif\n" + old)
src = re.sub(r"weyl_mix\((\w+), (n[01]\.[xy]), p\)", r"weyl_mix(\1, \2, p, pl.mg)", src)
src = re.sub(r"weyl_mix\((\w+ \+ p\.omega), (n[01]\.[xy]), p\)", r"weyl_mix(\1, \2, p, pl.mg)", src)
open(d + "/xg_pairs.cuh", "w").write(src)
out = f"{PKG}/lib/alt/libxg_gpu_{name}.so"; os.makedirs(os.path.dirname(out), exist_ok=True)
cmd = ["/usr/local/cuda/bin/nvcc", "-O3", "-std=c++17", "-gencode", "arch=compute_100a,code=sm_100a", "-lineinfo",
       "-Xcompiler", "-fPIC", "-shared", "-cudart", "static", "-I", ROOT + "/include", *[f"-D{x}" for x in defs],
       "-o", out, d + "/xg_gpu.cu"]
r = subprocess.run(cmd, capture_output=True, text=True); print(r.stdout[-3000:], r.stderr[-3000:]); sys.exit(r.returncode)
