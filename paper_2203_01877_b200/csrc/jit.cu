// jit.cu -- the dense group-by kernel compiled for one aggregation plan (NVRTC, sm_100a).
//
// The generic dense kernel (groupby.cu, gb_dense_kernel) interprets the plan at run time:
// per 4-row group it loops over the (op, expression) pairs and their factors, reads each
// factor's stage offset, constant and sign from kernel parameters and branches on them.
// Here the plan -- predicate terms, key columns, every pair's op and factors with their
// constants, the stage layout -- is written into CUDA source as literals, compiled once
// per distinct plan with NVRTC (libnvrtc is opened at run time) and loaded with the
// runtime's library API; each staged column is read from shared memory once per tile and
// every loop is straight-line code. The TMA stage pipeline, the lane-private
// accumulators, the exactness bound and the partial records are the generic kernel's
// (same arithmetic, same fixed slots, same direct merge), so the result is bit-identical;
// a compile failure or TQP_JIT=0 keeps the generic kernel. This is query compilation,
// TQP's own theme (SQL compiled into tensor programs), one level lower:
// the tensor program's aggregation kernel compiled for the query's expressions.
#include <dlfcn.h>

#include <sstream>
#include <vector>

#include "internal.h"
#include "jit.h"

#define TQP_JIT_STR(...) #__VA_ARGS__
#define TQP_JIT_XSTR(...) TQP_JIT_STR(__VA_ARGS__)

namespace tqp {

namespace {

// ------------------------------------------------------------- NVRTC, opened lazily
typedef int nvrtcRes;
typedef struct _nvrtcProgram* nvrtcProg;
struct Nvrtc {
    bool ok = false;
    nvrtcRes (*create)(nvrtcProg*, const char*, const char*, int, const char* const*, const char* const*) = nullptr;
    nvrtcRes (*compile)(nvrtcProg, int, const char* const*) = nullptr;
    nvrtcRes (*cubin_size)(nvrtcProg, size_t*) = nullptr;
    nvrtcRes (*cubin)(nvrtcProg, char*) = nullptr;
    nvrtcRes (*log_size)(nvrtcProg, size_t*) = nullptr;
    nvrtcRes (*log)(nvrtcProg, char*) = nullptr;
    nvrtcRes (*destroy)(nvrtcProg*) = nullptr;
};

Nvrtc& nvrtc() {
    static Nvrtc n = [] {
        Nvrtc r;
        void* h = dlopen("libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("/usr/local/cuda/lib64/libnvrtc.so.12", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return r;
        r.create = (decltype(r.create))dlsym(h, "nvrtcCreateProgram");
        r.compile = (decltype(r.compile))dlsym(h, "nvrtcCompileProgram");
        r.cubin_size = (decltype(r.cubin_size))dlsym(h, "nvrtcGetCUBINSize");
        r.cubin = (decltype(r.cubin))dlsym(h, "nvrtcGetCUBIN");
        r.log_size = (decltype(r.log_size))dlsym(h, "nvrtcGetProgramLogSize");
        r.log = (decltype(r.log))dlsym(h, "nvrtcGetProgramLog");
        r.destroy = (decltype(r.destroy))dlsym(h, "nvrtcDestroyProgram");
        r.ok = r.create && r.compile && r.cubin_size && r.cubin && r.log_size && r.log && r.destroy;
        return r;
    }();
    return n;
}

// the generated translation unit's fixed part: types, the parameter block, TMA helpers
const char* kPrelude =
    "typedef unsigned long long u64; typedef long long i64; typedef unsigned int u32; typedef unsigned char u8;\n"
    "struct JA " TQP_JIT_XSTR(TQP_DENSE_JIT_ARGS_BODY) ";\n"
    R"(
__device__ __forceinline__ u32 smem_u32(const void* p) { return (u32)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(u64* bar, u32 c) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(c) : "memory"); }
__device__ __forceinline__ void fence_mbar_init() { asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory"); }
__device__ __forceinline__ void fence_proxy_async() { asm volatile("fence.proxy.async.shared::cta;" ::: "memory"); }
__device__ __forceinline__ void mbar_expect_tx(u64* bar, u32 b) {
    asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(b) : "memory"); }
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, u32 bytes, u64* bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                 ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory"); }
__device__ __forceinline__ void mbar_wait(u64* bar, u32 parity) {
    asm volatile("{\n .reg .pred p;\n WAIT_%=:\n mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n @!p bra WAIT_%=;\n}\n"
                 ::"r"(smem_u32(bar)), "r"(parity) : "memory"); }
)";

std::string u64lit(unsigned long long v) {
    std::ostringstream o;
    o << v << "ull";
    return o.str();
}
const char* ctype(int dt) { return dt == TQP_U8 ? "u8" : dt == TQP_I32 ? "int" : "i64"; }
int esize(int dt) { return dt == TQP_U8 ? 1 : dt == TQP_I32 ? 4 : 8; }

// Rows of a thread in the tile: paired (default) = rows 2 tid, 2 tid + 1, 2 NT + 2 tid,
// 2 NT + 2 tid + 1, so each shared-memory vector load of a warp is contiguous (no bank
// conflicts); else 4 tid .. 4 tid + 3 (lanes 32 bytes apart in an int64 column: 2-way
// conflicts on every 16-byte load). Aggregation does not care which thread takes a row.
#ifndef TQP_JIT_PAIRED
#define TQP_JIT_PAIRED 1
#endif

// the 4 rows of stage slot u for this thread, sign / zero extended: x<u>_<i>
void emit_load(std::ostringstream& o, const DenseJitSpec& s, int u) {
    const int off = s.uoff[u];
    if (TQP_JIT_PAIRED) {
        const int NT = s.nt;
        if (s.udt[u] == TQP_I64) {
            o << "      const longlong2 a" << u << " = reinterpret_cast<const longlong2*>(st + " << off << ")[tid];\n"
              << "      const longlong2 b" << u << " = reinterpret_cast<const longlong2*>(st + " << off << ")[" << NT << " + tid];\n"
              << "      const i64 x" << u << "_0 = a" << u << ".x, x" << u << "_1 = a" << u << ".y, x" << u << "_2 = b" << u
              << ".x, x" << u << "_3 = b" << u << ".y;\n";
        } else if (s.udt[u] == TQP_I32) {
            o << "      const int2 a" << u << " = reinterpret_cast<const int2*>(st + " << off << ")[tid];\n"
              << "      const int2 b" << u << " = reinterpret_cast<const int2*>(st + " << off << ")[" << NT << " + tid];\n"
              << "      const i64 x" << u << "_0 = a" << u << ".x, x" << u << "_1 = a" << u << ".y, x" << u << "_2 = b" << u
              << ".x, x" << u << "_3 = b" << u << ".y;\n";
        } else {
            o << "      const u32 a" << u << " = reinterpret_cast<const unsigned short*>(st + " << off << ")[tid];\n"
              << "      const u32 b" << u << " = reinterpret_cast<const unsigned short*>(st + " << off << ")[" << NT << " + tid];\n"
              << "      const i64 x" << u << "_0 = (i64)(a" << u << " & 0xFFu), x" << u << "_1 = (i64)(a" << u << " >> 8), x" << u
              << "_2 = (i64)(b" << u << " & 0xFFu), x" << u << "_3 = (i64)(b" << u << " >> 8);\n";
        }
        return;
    }
    if (s.udt[u] == TQP_I64) {
        o << "      const longlong2 a" << u << " = reinterpret_cast<const longlong2*>(st + " << off << ")[2 * tid];\n"
          << "      const longlong2 b" << u << " = reinterpret_cast<const longlong2*>(st + " << off << ")[2 * tid + 1];\n"
          << "      const i64 x" << u << "_0 = a" << u << ".x, x" << u << "_1 = a" << u << ".y, x" << u << "_2 = b" << u
          << ".x, x" << u << "_3 = b" << u << ".y;\n";
    } else if (s.udt[u] == TQP_I32) {
        o << "      const int4 a" << u << " = reinterpret_cast<const int4*>(st + " << off << ")[tid];\n"
          << "      const i64 x" << u << "_0 = a" << u << ".x, x" << u << "_1 = a" << u << ".y, x" << u << "_2 = a" << u
          << ".z, x" << u << "_3 = a" << u << ".w;\n";
    } else {
        o << "      const u32 a" << u << " = reinterpret_cast<const u32*>(st + " << off << ")[tid];\n";
        for (int i = 0; i < 4; i++)
            o << "      const i64 x" << u << "_" << i << " = (i64)((a" << u << " >> " << 8 * i << ") & 0xFFu);\n";
    }
}

}  // namespace

std::string dense_jit_source(const DenseJitSpec& s) {
    std::ostringstream o;
    const int NT = s.nt, NS = s.ns, NP = s.n_pairs, NK = s.n_keys, TR = NT * 4, SB = s.stage_bytes;
    auto X = [](int u, int i) { return "x" + std::to_string(u) + "_" + std::to_string(i); };
    o << kPrelude;
    o << "extern \"C\" __global__ void __launch_bounds__(" << NT << ") tqp_groupby_dense_jit(JA a) {\n"
      << "  extern __shared__ __align__(128) u8 smem[];\n"
      << "  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;\n"
      << "  const int D = a.D;\n"
      << "  u64* const mbar = reinterpret_cast<u64*>(smem + " << NS * SB << ");\n"
      << "  u64* const kmin = mbar + 4;\n"
      << "  int* const kshift = reinterpret_cast<int*>(kmin + 8);\n"
      << "  i64* const dcnt = reinterpret_cast<i64*>(kshift + 8);\n"
      << "  int* const bad = reinterpret_cast<int*>(dcnt + 16);\n"
      << "  i64* const acc = reinterpret_cast<i64*>(smem + " << NS * SB + DENSE_JIT_HDR << ");\n"
      << "  u32* const cnt = reinterpret_cast<u32*>(acc + (i64)D * " << NP * NT << ");\n";
    // accumulators (own column only: no barrier needed before use)
    o << "  for (int d = 0; d < D; d++) {\n    cnt[d * " << NT << " + tid] = 0;\n";
    for (int j = 0; j < NP; j++)
        o << "    acc[(i64)(d * " << NP << " + " << j << ") * " << NT << " + tid] = "
          << (s.prop[j] == 0 ? "0" : s.prop[j] == 1 ? "9223372036854775807ll" : "(-9223372036854775807ll - 1)") << ";\n";
    o << "  }\n";
    // header: mbarriers, the packed-key layout from the device-resident key ranges
    o << "  if (tid == 0) {\n";
    for (int st = 0; st < NS; st++) o << "    mbar_init(&mbar[" << st << "], 1);\n";
    o << "    fence_mbar_init();\n    int off = 0;\n";
    for (int k = NK - 1; k >= 0; k--)
        o << "    { const u64 mn = a.krange[" << k << "], mx = a.krange[" << 8 + k << "];\n"
          << "      const int w = mx > mn ? 64 - __clzll(mx - mn) : 0;\n"
          << "      kmin[" << k << "] = mx >= mn ? mn : 0; kshift[" << k << "] = off; off += w; }\n";
    o << "    *bad = 0;\n  }\n  __syncthreads();\n";
    if (s.dk)
        o << "  const u32 dk0 = 0 < D ? (u32)a.dkeys[0] : 0xFFFFFFFFu, dk1 = 1 < D ? (u32)a.dkeys[1] : 0xFFFFFFFFu;\n"
          << "  const u32 dk2 = 2 < D ? (u32)a.dkeys[2] : 0xFFFFFFFFu, dk3 = 3 < D ? (u32)a.dkeys[3] : 0xFFFFFFFFu;\n";
    for (int k = 0; k < NK; k++) o << "  const u64 km" << k << " = kmin[" << k << "];\n  const int ks" << k << " = kshift[" << k << "];\n";
    // per (pair, own factor): OR of |add +- x| over every staged row (the bound argument)
    for (int j = 0; j < NP; j++)
        for (int f = s.pext[j]; f < s.pnf[j]; f++) o << "  u64 mt" << j << "_" << f << " = 0;\n";
    o << "  u32 wpar = 0;\n  bool unseen = false;\n";
    o << "  auto eligible = [&](i64 t) { return a.bulk_ok && (t + 1) * " << TR << " <= a.n; };\n";
    o << "  auto issue = [&](i64 t, int s) {\n    mbar_expect_tx(&mbar[s], " << SB << ");\n";
    for (int u = 0; u < s.n_ucols; u++)
        o << "    bulk_g2s(smem + s * " << SB << " + " << s.uoff[u] << ", (const u8*)a.ucol[" << u << "] + t * "
          << TR * esize(s.udt[u]) << ", " << TR * esize(s.udt[u]) << ", &mbar[s]);\n";
    o << "  };\n";
    o << "  if (tid == 0)\n    for (int s = 0; s < " << NS << "; s++) {\n"
      << "      const i64 t = blockIdx.x + (i64)s * gridDim.x;\n"
      << "      if (t < a.n_tiles && eligible(t)) issue(t, s);\n    }\n";
    o << "  for (i64 k = 0;; k++) {\n"
      << "    const i64 t = blockIdx.x + k * gridDim.x;\n    if (t >= a.n_tiles) break;\n"
      << "    const int s = " << (NS == 1 ? "0" : "(int)(k % " + std::to_string(NS) + ")") << ";\n"
      << "    const u8* const st = smem + s * " << SB << ";\n"
      << "    const int nrows = (int)min((i64)" << TR << ", a.n - t * " << TR << ");\n"
      << "    if (eligible(t)) {\n      mbar_wait(&mbar[s], (wpar >> s) & 1u);\n      wpar ^= 1u << s;\n    } else {\n";
    for (int u = 0; u < s.n_ucols; u++) {
        const char* ct = ctype(s.udt[u]);
        o << "      for (int r = tid; r < " << TR << "; r += " << NT << ") reinterpret_cast<" << ct << "*>(smem + s * "
          << SB << " + " << s.uoff[u] << ")[r] = r < nrows ? ((const " << ct << "*)a.ucol[" << u << "])[t * " << TR
          << " + r] : (" << ct << ")0;\n";
    }
    o << "      __syncthreads();\n    }\n";
    // ---- one tile: 4 consecutive rows per thread
    if (TQP_JIT_PAIRED) {
        o << "    {\n";
        for (int i = 0; i < 4; i++)
            o << "      bool p" << i << " = " << (s.never ? "false && " : "") << "(" << (i < 2 ? 0 : 2 * NT) << " + 2 * tid + "
              << (i & 1) << ") < nrows;\n";
    } else {
        o << "    {\n      const int r0 = tid * 4;\n";
        for (int i = 0; i < 4; i++) o << "      bool p" << i << " = " << (s.never ? "false && " : "") << "r0 + " << i << " < nrows;\n";
    }
    std::vector<bool> used(s.n_ucols, false);
    for (int q = 0; q < s.n_terms; q++) used[s.tcol[q]] = true;
    for (int k = 0; k < NK; k++) used[s.kslot[k]] = true;
    for (int j = 0; j < NP; j++)
        for (int f = s.pext[j]; f < s.pnf[j]; f++) used[s.pslot[j][f]] = true;
    for (int u = 0; u < s.n_ucols; u++)
        if (used[u]) emit_load(o, s, u);
    for (int q = 0; q < s.n_terms; q++) {
        const int u = s.tcol[q];
        for (int i = 0; i < 4; i++) {
            if (s.tdt[q] == TQP_I64)
                o << "      p" << i << " = p" << i << " && (((u64)" << X(u, i) << " - " << u64lit(s.tlo[q]) << " <= "
                  << u64lit(s.twidth[q]) << ") != " << (s.tneg[q] ? "true" : "false") << ");\n";
            else
                o << "      p" << i << " = p" << i << " && (((u32)" << X(u, i) << " - " << (unsigned)(uint32_t)s.tlo[q]
                  << "u <= " << (unsigned)(uint32_t)s.twidth[q] << "u) != " << (s.tneg[q] ? "true" : "false") << ");\n";
        }
    }
    o << "      if (p0 | p1 | p2 | p3) {\n";
    for (int i = 0; i < 4; i++) {   // packed key -> dense id
        o << "        const u32 kb" << i << " = 0u";
        for (int k = 0; k < NK; k++) {
            const int u = s.kslot[k];
            std::string part = s.udt[u] == TQP_U8    ? "(u64)" + X(u, i)
                               : s.udt[u] == TQP_I32 ? "(u64)((u32)" + X(u, i) + " ^ 0x80000000u)"
                                                     : "((u64)" + X(u, i) + " ^ 0x8000000000000000ull)";
            o << " | ((u32)(" << part << " - km" << k << ") << ks" << k << ")";
        }
        o << ";\n";
        if (s.dk)
            o << "        int id" << i << " = (dk0 < kb" << i << ") + (dk1 < kb" << i << ") + (dk2 < kb" << i << ") + (dk3 < kb"
              << i << ");\n        if (!(dk0 == kb" << i << " || dk1 == kb" << i << " || dk2 == kb" << i << " || dk3 == kb" << i
              << ")) id" << i << " = 16;\n        if (!p" << i << ") id" << i << " = 0;\n";
        else
            o << "        const int id" << i << " = p" << i << " ? (int)__ldg(a.dtab + kb" << i << ") : 0;\n";
        o << "        if (id" << i << " >= D) { unseen = true; p" << i << " = false; }\n"
          << "        if (p" << i << ") cnt[id" << i << " * " << NT << " + tid]++;\n";
    }
    // every pair: value = product of its factors (a pair extending the previous pair's
    // factor list starts from that pair's value), wrapped 64-bit arithmetic
    for (int j = 0; j < NP; j++) {
        for (int i = 0; i < 4; i++) {
            std::string v = "v" + std::to_string(j) + "_" + std::to_string(i);
            o << "        i64 " << v << " = " << (s.pext[j] ? "v" + std::to_string(j - 1) + "_" + std::to_string(i) : "1") << ";\n";
            for (int f = s.pext[j]; f < s.pnf[j]; f++) {
                o << "        { const i64 tt = (i64)(" << u64lit((unsigned long long)s.padd[j][f])
                  << (s.psign[j][f] < 0 ? " - " : " + ") << "(u64)" << X(s.pslot[j][f], i) << ");\n"
                  << "          mt" << j << "_" << f << " |= (u64)(tt ^ (tt >> 63));\n"
                  << "          " << v << " = " << (f == 0 ? std::string("tt") : "(i64)((u64)" + v + " * (u64)tt)") << "; }\n";
            }
        }
        for (int i = 0; i < 4; i++) {
            const std::string v = "v" + std::to_string(j) + "_" + std::to_string(i);
            o << "        if (p" << i << ") { i64* const pa = acc + (i64)(id" << i << " * " << NP << " + " << j << ") * " << NT
              << " + tid; ";
            if (s.prop[j] == 0) o << "*pa += " << v << "; }\n";
            else if (s.prop[j] == 1) o << "*pa = min(*pa, " << v << "); }\n";
            else o << "*pa = max(*pa, " << v << "); }\n";
        }
    }
    o << "      }\n    }\n";
    o << "    __syncthreads();\n"
      << "    const i64 t2 = t + (i64)" << NS << " * gridDim.x;\n"
      << "    if (tid == 0 && t2 < a.n_tiles && eligible(t2)) { fence_proxy_async(); issue(t2, s); }\n  }\n";
    o << "  if (unseen) atomicOr(a.overflow, 8);\n";
    // exactness bound per pair: sum of its factors' bit lengths (a shared factor's bound is
    // the pair's that computed it)
    o << "  bool badv = false;\n";
    for (int j = 0; j < NP; j++) {
        o << "  { int bs = 0;\n";
        for (int f = 0; f < s.pnf[j]; f++) {
            int jj = j;
            while (f < s.pext[jj]) jj--;
            o << "    bs += 64 - __clzll(mt" << jj << "_" << f << ");\n";
        }
        o << "    badv |= bs > " << (s.prop[j] == 0 ? "a.dense_bits" : "62") << "; }\n";
    }
    o << "  if (badv) *bad = 1;\n";
    // flush: counts per id, one partial record per (CTA, id) at the fixed slot blockIdx.x * D + id
    o << "  for (int d = warp; d < D; d += " << NT / 32 << ") {\n"
      << "    i64 c = 0;\n    for (int t2 = lane; t2 < " << NT << "; t2 += 32) c += cnt[d * " << NT << " + t2];\n"
      << "    for (int o2 = 16; o2 > 0; o2 >>= 1) c += __shfl_xor_sync(0xffffffffu, c, o2);\n"
      << "    if (lane == 0) dcnt[d] = c;\n  }\n  __syncthreads();\n"
      << "  if (tid == 0 && *bad) atomicOr(a.overflow, 4);\n"
      << "  for (int s2 = warp; s2 < D * " << NP << "; s2 += " << NT / 32 << ") {\n"
      << "    const int d = s2 / " << NP << ", jj = s2 - d * " << NP << ";\n"
      << "    const i64 rec = (i64)blockIdx.x * D + d;\n"
      << "    const i64* col = acc + (i64)s2 * " << NT << ";\n"
      << "    const int op = ";
    for (int j = 0; j < NP; j++) o << "jj == " << j << " ? " << s.prop[j] << " : ";
    o << "0;\n"
      << "    if (op == 0) {   // exact: split halves of the per-thread int64 sums\n"
      << "      u64 lo = 0; i64 hi = 0;\n"
      << "      for (int t2 = lane; t2 < " << NT << "; t2 += 32) { lo += (u64)(u32)col[t2]; hi += col[t2] >> 32; }\n"
      << "      for (int o2 = 16; o2 > 0; o2 >>= 1) { lo += __shfl_xor_sync(0xffffffffu, lo, o2); hi += __shfl_xor_sync(0xffffffffu, hi, o2); }\n"
      << "      if (lane == 0) { a.plo[jj][rec] = lo; a.phi[jj][rec] = hi; }\n"
      << "    } else {\n      i64 v = op == 1 ? 9223372036854775807ll : (-9223372036854775807ll - 1);\n"
      << "      for (int t2 = lane; t2 < " << NT << "; t2 += 32) v = op == 1 ? min(v, col[t2]) : max(v, col[t2]);\n"
      << "      for (int o2 = 16; o2 > 0; o2 >>= 1) { const i64 y = __shfl_xor_sync(0xffffffffu, v, o2); v = op == 1 ? min(v, y) : max(v, y); }\n"
      << "      if (lane == 0) a.plo[jj][rec] = (u64)v;\n    }\n  }\n"
      << "  for (int d = tid; d < D; d += " << NT << ") {\n"
      << "    const i64 rec = (i64)blockIdx.x * D + d;\n    a.pkey[rec] = a.dkeys[d];\n    a.pcount[rec] = dcnt[d];\n  }\n"
      << "}\n";
    return o.str();
}

namespace {
struct JitKernel {
    cudaLibrary_t lib = nullptr;
    cudaKernel_t k = nullptr;
    std::map<int, size_t> smem_set;   // per device: the dynamic shared memory limit set so far
    std::map<size_t, int> occ;        // resident CTAs per SM by dynamic shared memory bytes
};
std::mutex& jit_mutex() {
    static std::mutex m;
    return m;
}
JitCounters g_counters;   // guarded by jit_mutex
std::map<std::string, JitKernel>& jit_cache() {
    static std::map<std::string, JitKernel> c;
    return c;
}

// the compiled kernel for the plan (cached by the plan's bytes -- the caller zero-fills the
// spec, padding included -- so a hit costs no source generation); null when unavailable
JitKernel* dense_jit_kernel(const DenseJitSpec& s) {
    std::string key(reinterpret_cast<const char*>(&s), sizeof(s));
    std::lock_guard<std::mutex> g(jit_mutex());
    auto& cache = jit_cache();
    auto it = cache.find(key);
    if (it != cache.end()) return it->second.k ? &it->second : nullptr;
    // a bounded number of compiled plans per process (each holds a loaded module); past it,
    // new plans run on the generic kernel
    constexpr size_t MAX_PLANS = 256;
    if (cache.size() >= MAX_PLANS) return nullptr;
    const std::string src = dense_jit_source(s);
    JitKernel jk;
    Nvrtc& nv = nvrtc();
    nvrtcProg prog = nullptr;
    if (nv.ok && nv.create(&prog, src.c_str(), "tqp_groupby_dense_jit.cu", 0, nullptr, nullptr) == 0) {
        const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo"};
        if (nv.compile(prog, 3, opts) == 0) {
            size_t n = 0;
            nv.cubin_size(prog, &n);
            std::string cubin(n, '\0');
            nv.cubin(prog, &cubin[0]);
            if (cudaLibraryLoadData(&jk.lib, cubin.data(), nullptr, nullptr, 0, nullptr, nullptr, 0) != cudaSuccess ||
                cudaLibraryGetKernel(&jk.k, jk.lib, "tqp_groupby_dense_jit") != cudaSuccess) {
                cudaGetLastError();
                jk.k = nullptr;
                fprintf(stderr, "libtqp: loading the compiled dense group-by kernel failed (generic kernel used)\n");
            }
        } else {
            size_t ln = 0;
            nv.log_size(prog, &ln);
            std::string log(ln, '\0');
            if (ln) nv.log(prog, &log[0]);
            fprintf(stderr, "libtqp: compiling the dense group-by kernel failed (generic kernel used):\n%s\n",
                    log.substr(0, 4000).c_str());
        }
        nv.destroy(&prog);
    }
    (jk.k ? g_counters.compiled : g_counters.failed)++;
    auto& slot = cache[std::move(key)];
    slot = jk;
    return slot.k ? &slot : nullptr;
}

bool set_jit_smem(JitKernel* jk, size_t smem) {
    int dev = 0;
    if (cudaGetDevice(&dev) != cudaSuccess) return false;
    size_t& cur = jk->smem_set[dev];
    if (smem <= cur) return true;
    if (cudaFuncSetAttribute((const void*)jk->k, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess) {
        cudaGetLastError();
        return false;
    }
    cur = smem;
    return true;
}
}  // namespace

bool jit_available() { return nvrtc().ok; }

JitCounters jit_counters() {
    std::lock_guard<std::mutex> g(jit_mutex());
    return g_counters;
}

bool jit_enabled() {
    const char* e = std::getenv("TQP_JIT");
    if (e && e[0] == '0') return false;
    return nvrtc().ok;
}

int dense_jit_occupancy(const DenseJitSpec& s, size_t smem) {
    JitKernel* jk = dense_jit_kernel(s);
    if (!jk) return 0;
    std::lock_guard<std::mutex> g(jit_mutex());
    auto it = jk->occ.find(smem);
    if (it != jk->occ.end()) return it->second;
    if (!set_jit_smem(jk, smem)) return 0;
    int occ = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, (const void*)jk->k, s.nt, smem) != cudaSuccess) {
        cudaGetLastError();
        return 0;
    }
    jk->occ[smem] = occ;
    return occ;
}

bool dense_jit_launch(tqp_ctx* ctx, const DenseJitSpec& s, const DenseJitArgs& args, int64_t grid, size_t smem,
                      const char* name) {
    JitKernel* jk = dense_jit_kernel(s);
    if (!jk) return false;
    {
        std::lock_guard<std::mutex> g(jit_mutex());
        if (!set_jit_smem(jk, smem)) return false;
    }
    cudaEvent_t a = nullptr, b = nullptr;
    const bool prof = ctx->profiled(name);
    if (prof) {
        a = ctx->get_event();
        b = ctx->get_event();
        TQP_CUDA(cudaEventRecord(a, ctx->stream));
    }
    DenseJitArgs ja = args;
    void* params[] = {&ja};
    const cudaError_t e = cudaLaunchKernel((const void*)jk->k, dim3((unsigned)grid), dim3(s.nt), params, smem, ctx->stream);
    if (e != cudaSuccess) fail(TQP_ERR_CUDA, std::string("launch ") + name + " (compiled): " + cudaGetErrorString(e));
    ctx->launches++;
    {
        std::lock_guard<std::mutex> g(jit_mutex());
        g_counters.launches++;
    }
    if (prof) {
        TQP_CUDA(cudaEventRecord(b, ctx->stream));
        ctx->pending.push_back({name, a, b});
    }
    return true;
}

}  // namespace tqp
