// tools/jit_check.cu -- generate the compiled dense group-by kernel's source for a TPC-H
// Q1-shaped plan and compile it with NVRTC (no GPU needed); prints the source with
// --print, writes the cubin for cuobjdump / nvdisasm with --cubin PATH.
//   nvcc -std=c++17 -I paper_2203_01877_b200/csrc tools/jit_check.cu -o /tmp/jit_check \
//        -L paper_2203_01877_b200 -ltqp -lnvrtc -Xlinker -rpath=$PWD/paper_2203_01877_b200
#include <nvrtc.h>

#include <cstdio>
#include <cstring>
#include <fstream>

#include "jit.h"

int main(int argc, char** argv) {
    using namespace tqp;
    DenseJitSpec s;
    // Q1: slots 0 shipdate i32, 1 returnflag u8, 2 linestatus u8, 3 quantity, 4 extendedprice,
    // 5 discount, 6 tax (i64 fixed point); NT = 128 -> 512 rows per stage
    const int dts[7] = {TQP_I32, TQP_U8, TQP_U8, TQP_I64, TQP_I64, TQP_I64, TQP_I64};
    int off = 0;
    s.n_ucols = 7;
    for (int u = 0; u < 7; u++) {
        s.udt[u] = dts[u];
        s.uoff[u] = off;
        off += 512 * (dts[u] == TQP_U8 ? 1 : dts[u] == TQP_I32 ? 4 : 8);
    }
    s.stage_bytes = off;
    s.n_terms = 1;
    s.tcol[0] = 0; s.tdt[0] = TQP_I32; s.tneg[0] = 0; s.tlo[0] = (unsigned)INT32_MIN; s.twidth[0] = 10471ull - INT32_MIN;
    s.n_keys = 2; s.kslot[0] = 1; s.kslot[1] = 2;
    s.n_pairs = 6;
    // sum(qty), sum(price), sum(price * (1 - disc)), sum(price * (1 - disc) * (1 + tax)), sum(disc), max(qty)
    s.prop[0] = 0; s.pnf[0] = 1; s.pslot[0][0] = 3; s.psign[0][0] = 1;
    s.prop[1] = 0; s.pnf[1] = 1; s.pslot[1][0] = 4; s.psign[1][0] = 1;
    s.prop[2] = 0; s.pnf[2] = 2; s.pext[2] = 1; s.pslot[2][0] = 4; s.psign[2][0] = 1; s.pslot[2][1] = 5; s.psign[2][1] = -1; s.padd[2][1] = 100;
    s.prop[3] = 0; s.pnf[3] = 3; s.pext[3] = 2; s.pslot[3][0] = 4; s.psign[3][0] = 1; s.pslot[3][1] = 5; s.psign[3][1] = -1; s.padd[3][1] = 100;
    s.pslot[3][2] = 6; s.psign[3][2] = 1; s.padd[3][2] = 100;
    s.prop[4] = 0; s.pnf[4] = 1; s.pslot[4][0] = 5; s.psign[4][0] = 1;
    s.prop[5] = 2; s.pnf[5] = 1; s.pslot[5][0] = 3; s.psign[5][0] = 1;
    s.dk = 4;
    const std::string src = dense_jit_source(s);
    const char* cubin_path = nullptr;
    for (int i = 1; i < argc; i++) {
        if (!strcmp(argv[i], "--print")) fputs(src.c_str(), stdout);
        if (!strcmp(argv[i], "--cubin") && i + 1 < argc) cubin_path = argv[i + 1];
        if (!strcmp(argv[i], "--dk0")) s.dk = 0;
    }
    nvrtcProgram p;
    nvrtcCreateProgram(&p, src.c_str(), "q1.cu", 0, nullptr, nullptr);
    const char* opts[] = {"-arch=sm_100a", "-std=c++17", "-lineinfo"};
    const nvrtcResult r = nvrtcCompileProgram(p, 3, opts);
    size_t ln = 0;
    nvrtcGetProgramLogSize(p, &ln);
    std::string log(ln, '\0');
    nvrtcGetProgramLog(p, &log[0]);
    fprintf(stderr, "compile: %s\n%s\n", nvrtcGetErrorString(r), log.c_str());
    if (r != NVRTC_SUCCESS) return 1;
    size_t n = 0;
    nvrtcGetCUBINSize(p, &n);
    std::string cubin(n, '\0');
    nvrtcGetCUBIN(p, &cubin[0]);
    if (cubin_path) std::ofstream(cubin_path, std::ios::binary).write(cubin.data(), n);
    fprintf(stderr, "cubin: %zu bytes\n", n);
    return 0;
}
