// jit.h -- JIT-specialized fused struct-for kernels (jit.cpp).
#pragma once
#include <stdint.h>
#include "sg_internal.h"

namespace sg {

// The content of one fused struct-for group: what the specialized kernel is
// compiled for (and hashed by).
struct JitGroup {
  int nops = 0;
  int nd = 0;     // quad-path dimensionality (0: generic cell path)
  int gl = 0;     // constant block geometry (0: runtime)
  int i32 = 0;    // value type int (else float)
  int stream = 0; // 8^3 streaming structure (stream8_body) instead of the tile loop
  DOp ops[SG_MAXOPS];
};

uint64_t jit_key(const JitGroup& g);
bool jit_group_of(const DTree& t, const DOp* ops, int nops, JitGroup& g);   // kernels.cu
// The specialized kernel of g's content (a cudaKernel_t usable with
// cudaLaunchKernel), or null while it compiles / when the JIT is off.
// prefetch: submit the compile without waiting even in synchronous mode (a
// flush submits every group of its plan first: they compile in parallel).
const void* jit_lookup(const JitGroup& g, bool prefetch = false);
// Bumped whenever a specialized kernel becomes ready (CUDA-graph signatures).
int64_t jit_generation();
void jit_set_mode(int m);   // -1: back to SG_JIT
void jit_shutdown();        // drop queued compiles, wait for in-flight ones, JIT off for good
int jit_selftest(int nd, int gl, int i32, const int32_t* ops, int nops, char* log, int64_t cap);
// [mode, ready, pending, failed, hits, misses, compile_us_total]
void jit_stats(int64_t* out, int n);

}  // namespace sg
