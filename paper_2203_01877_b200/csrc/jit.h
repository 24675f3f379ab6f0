// jit.h -- the dense group-by kernel compiled per aggregation plan at run time (jit.cu).
#pragma once

#include <string>

#include "common.cuh"

// Kernel parameter block of the compiled kernel: one definition, compiled into libtqp and
// pasted (stringified) into the generated source, so both sides share the layout.
#define TQP_DENSE_JIT_ARGS_BODY                                                                         \
    {                                                                                                   \
        const void* ucol[16];                                                                           \
        long long n;                                                                                    \
        long long n_tiles;                                                                              \
        int D;                                                                                          \
        int dense_bits;                                                                                 \
        int bulk_ok;                                                                                    \
        const unsigned long long* krange;                                                               \
        const unsigned long long* dkeys;                                                                \
        const unsigned char* dtab;                                                                      \
        int* overflow;                                                                                  \
        unsigned long long* plo[16];                                                                    \
        long long* phi[16];                                                                             \
        unsigned long long* pkey;                                                                       \
        long long* pcount;                                                                              \
    }

namespace tqp {

struct DenseJitArgs TQP_DENSE_JIT_ARGS_BODY;

// Everything the generated source fixes as literals (groupby.cu's Phase1Args, dense part).
// Compiled kernels are cached by the struct's bytes: zero-fill it (memset) before filling
// it in, so the padding is deterministic.
struct DenseJitSpec {
    int nt = 128;            // threads per CTA (4 rows each per tile)
    int ns = 1;              // TMA stages
    int stage_bytes = 0;     // one stage: every referenced column's nt * 4 rows
    int n_ucols = 0;
    int udt[16] = {};
    int uoff[16] = {};       // byte offset of each column in a stage
    int n_terms = 0;         // predicate conjunction: one interval test per term
    bool never = false;
    int tcol[16] = {}, tdt[16] = {}, tneg[16] = {};
    unsigned long long tlo[16] = {}, twidth[16] = {};
    int n_keys = 0;
    int kslot[8] = {};       // stage slot of key column k (column 0 most significant)
    int n_pairs = 0;         // (op, expression) pairs; expression = product of (add +- column)
    int prop[8] = {}, pnf[8] = {}, pext[8] = {};
    int pslot[8][3] = {}, psign[8][3] = {};
    long long padd[8][3] = {};
    int dk = 0;              // 4: dense ids by compares against <= 4 keys in registers; 0: table
};
constexpr int DENSE_JIT_HDR = 384;   // shared-memory header bytes after the stages

bool jit_enabled();
bool jit_available();   // libnvrtc found
struct JitCounters { int64_t compiled = 0, failed = 0, launches = 0; };
JitCounters jit_counters();
std::string dense_jit_source(const DenseJitSpec& s);
// resident CTAs per SM of the compiled kernel (compiles on first use); 0 = not available
int dense_jit_occupancy(const DenseJitSpec& s, size_t smem);
// launch on ctx->stream under the profiling name `name`; false = not available (nothing launched)
bool dense_jit_launch(tqp_ctx* ctx, const DenseJitSpec& s, const DenseJitArgs& args, int64_t grid, size_t smem,
                      const char* name);

}  // namespace tqp
