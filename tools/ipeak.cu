// Integer-pipe microbenchmark: LOP3 issue rate by operand form (tools/, not shipped).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

#define L3(d, a, b, c, lut) asm volatile("lop3.b32 %0, %1, %2, %3, " #lut ";" : "=r"(d) : "r"(a), "r"(b), "r"(c))
#define L3I(d, a, b, imm, lut) asm volatile("lop3.b32 %0, %1, %2, " #imm ", " #lut ";" : "=r"(d) : "r"(a), "r"(b))
#define SHF(d, a, b) asm volatile("shf.l.wrap.b32 %0, %1, %2, 1;" : "=r"(d) : "r"(a), "r"(b))
#define MADHI(d, a, b, c) asm volatile("mad.hi.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c))
#define MADW(d, a, b) asm volatile("{.reg .u64 t; mul.wide.u32 t, %1, %2; cvt.u32.u64 %0, t; shr.u64 t, t, 32; cvt.u32.u64 %1, t;}" : "=r"(d), "+r"(a) : "r"(b))
#define MAD(d, a, b, c) asm volatile("mad.lo.u32 %0, %1, %2, %3;" : "=r"(d) : "r"(a), "r"(b), "r"(c))

template <int MODE>
__global__ void k(uint32_t* sink, int iters, uint32_t seed) {
  uint32_t r[16];
  for (int i = 0; i < 16; ++i) r[i] = seed * (i + 3) ^ threadIdx.x;
  uint32_t m = seed | 3;
  for (int it = 0; it < iters; ++it) {
#pragma unroll
    for (int j = 0; j < 16; ++j) {
      uint32_t& a = r[j];
      const uint32_t b = r[(j + 5) & 15], c = r[(j + 11) & 15];
      if (MODE == 0) L3(a, a, b, c, 0x96);
      if (MODE == 1) L3I(a, a, b, 0x5555, 0x96);
      if (MODE == 2) SHF(a, a, b);
      if (MODE == 3) { if (j & 1) L3(a, a, b, c, 0x96); else MAD(a, a, m, b); }
      if (MODE == 4) MAD(a, a, m, b);
      if (MODE == 6) MADHI(a, a, m, b);
      if (MODE == 7) { if (j & 1) L3(a, a, b, c, 0x96); else MADHI(a, a, m, b); }
      if (MODE == 8) { if ((j & 3) == 0) MADHI(a, a, m, b); else if ((j & 3) == 1) MAD(a, a, m, b); else L3(a, a, b, c, 0x96); }
      if (MODE == 9) { uint32_t lo; MADW(lo, a, m); a ^= lo; }
      if (MODE == 10) { if (j < 10) L3(a, a, b, c, 0x96); else if (j < 12) { uint32_t lo, t = a; MADW(lo, t, m); a = lo + t; } else MAD(a, a, m, b); }
      if (MODE == 11) { if (j == 3 || j == 11) { uint32_t lo, t = a; MADW(lo, t, m); a = lo; r[(j + 1) & 15] ^= t; } else if (j == 7) { MAD(a, a, m, b); } else L3(a, a, b, c, 0x96); }
      if (MODE == 12) { if (j == 3 || j == 11) SHF(a, a, b); else if (j == 7) {} else L3(a, a, b, c, 0x96); }
      if (MODE == 13) { if (j == 7) {} else L3(a, a, b, c, 0x96); }
      if (MODE == 14) { if (j == 3 || j == 11) { MADHI(a, a, m, b); } else if (j == 7) { MAD(a, a, m, b); } else L3(a, a, b, c, 0x96); }
      if (MODE == 5) { if ((j & 3) == 0) MAD(a, a, m, b); else L3(a, a, b, c, 0x96); }
    }
  }
  uint32_t x = 0;
  for (int i = 0; i < 16; ++i) x ^= r[i];
  if (x == 0x12345678u) sink[0] = x;
}

template <int MODE>
void run(const char* name) {
  uint32_t* sink;
  cudaMalloc(&sink, 4);
  int blocks = 148 * 8, threads = 256, iters = 4096;
  k<MODE><<<blocks, threads>>>(sink, 16, 1);
  cudaEvent_t a, b;
  cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  k<MODE><<<blocks, threads>>>(sink, iters, 1);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = double(blocks) * threads * iters * 16;
  printf("%-26s %8.2f Tops/s (lane-ops at 16 per iteration) %8.3f ms\n", name, ops / ms / 1e9, ms);
  cudaFree(sink);
}

int main() {
  run<0>("lop3 3-reg");
  run<1>("lop3 2-reg+imm");
  run<2>("shf.wrap");
  run<4>("imad");
  run<3>("lop3/imad 1:1");
  run<5>("lop3/imad 3:1");
  run<9>("imad.wide(+lop)");
  run<10>("10lop:2wide:4imad");
  run<13>("15 lop3 (of 16 slots)");
  run<12>("13lop:2shf (of 16)");
  run<11>("13lop+2x(wide+xor):1imad");
  run<14>("13lop:2imad.hi:1imad");
  run<6>("imad.hi");
  run<7>("lop3/imad.hi 1:1");
  run<8>("lop3:imad:imad.hi 2:1:1");
  return 0;
}
