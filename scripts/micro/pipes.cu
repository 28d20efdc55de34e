// Throughput microbenchmark of the integer/FP instructions the hash and the
// decision use (IMAD lo/hi/wide, LOP3, SHF, IADD3, FMUL, FMNMX, ISETP+SEL),
// in thread-instructions per clock per SM. Build: nvcc -arch=sm_100a -O3.
#include <cstdio>
#include <cuda_runtime.h>

#define CH 8
#define IT 4096

template <int OP>
__global__ void k(unsigned* out, unsigned a0, unsigned m) {
  unsigned r[CH];
#pragma unroll
  for (int c = 0; c < CH; ++c) r[c] = a0 + threadIdx.x * 7 + c;
  for (int i = 0; i < IT; ++i) {
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      if (OP == 0) asm volatile("mad.lo.u32 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(m), "r"(a0));
      if (OP == 1) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(m), "r"(a0));
      if (OP == 2) { unsigned long long w; asm volatile("mul.wide.u32 %0, %1, %2;" : "=l"(w) : "r"(r[c]), "r"(m)); r[c] = (unsigned)w ^ (unsigned)(w >> 32); }
      if (OP == 3) asm volatile("lop3.b32 %0, %0, %1, %2, 0x96;" : "+r"(r[c]) : "r"(m), "r"(a0));
      if (OP == 4) asm volatile("shf.r.clamp.b32 %0, %0, %1, 27;" : "+r"(r[c]) : "r"(m));
      if (OP == 5) asm volatile("add.u32 %0, %0, %1;" : "+r"(r[c]) : "r"(m));
      if (OP == 6) { float f = __uint_as_float(r[c]); asm volatile("mul.f32 %0, %0, %1;" : "+f"(f) : "f"(__uint_as_float(m))); r[c] = __float_as_uint(f); }
      if (OP == 7) { float f = __uint_as_float(r[c]); asm volatile("max.f32 %0, %0, %1;" : "+f"(f) : "f"(__uint_as_float(m))); r[c] = __float_as_uint(f); }
      if (OP == 8) asm volatile("mul.hi.u32 %0, %0, %1;" : "+r"(r[c]) : "r"(m));
      if (OP == 9) asm volatile("shr.u32 %0, %0, %1;" : "+r"(r[c]) : "r"(m));
      if (OP == 10) asm volatile("mul.lo.u32 %0, %0, %1;" : "+r"(r[c]) : "r"(m));
      if (OP == 11) { unsigned t; asm volatile("clz.b32 %0, %1;" : "=r"(t) : "r"(r[c])); r[c] ^= t + m; }
      if (OP == 12) asm volatile("prmt.b32 %0, %0, %1, 0x5140;" : "+r"(r[c]) : "r"(m));
      if (OP == 13) asm volatile("min.u32 %0, %0, %1;" : "+r"(r[c]) : "r"(m + c));
      if (OP == 14) { unsigned t; asm volatile("{.reg .pred p; setp.lt.u32 p, %1, %2; selp.u32 %0, %1, %2, p;}" : "=r"(t) : "r"(r[c]), "r"(m)); r[c] = t ^ a0; }
      if (OP == 15) { unsigned long long w = ((unsigned long long)m << 32) | a0; unsigned long long o; asm volatile("mad.wide.u32 %0, %1, %2, %3;" : "=l"(o) : "r"(r[c]), "r"(m), "l"(w)); r[c] = (unsigned)(o >> 32); }
      if (OP == 16) asm volatile("mad.hi.u32 %0, %0, %1, %2;" : "+r"(r[c]) : "r"(m), "r"(r[(c + 1) % CH]));
    }
  }
  unsigned acc = 0;
#pragma unroll
  for (int c = 0; c < CH; ++c) acc ^= r[c];
  if (acc == 0x12345678u) out[0] = acc;
}

template <int OP>
void run(const char* name, int sms, int clk_khz) {
  unsigned* out;
  cudaMalloc(&out, 4);
  const int blocks = sms * 8, threads = 256;
  k<OP><<<blocks, threads>>>(out, 3, 0x9e3779b9u);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaEventRecord(a);
  k<OP><<<blocks, threads>>>(out, 3, 0x9e3779b9u);
  cudaEventRecord(b);
  cudaEventSynchronize(b);
  float ms;
  cudaEventElapsedTime(&ms, a, b);
  const double ops = double(blocks) * threads * IT * CH;
  const double per_clk_sm = ops / (ms * 1e-3) / (clk_khz * 1e3) / sms;
  printf("%-10s %8.3f ms  %7.1f thread-ops/clk/SM\n", name, ms, per_clk_sm);
  cudaFree(out);
}

int main() {
  int sms, clk;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  printf("SMs %d clock %d kHz\n", sms, clk);
  run<0>("imad.lo", sms, clk);
  run<10>("mul.lo", sms, clk);
  run<1>("imad.hi", sms, clk);
  run<8>("mul.hi", sms, clk);
  run<2>("mul.wide+x", sms, clk);
  run<3>("lop3", sms, clk);
  run<4>("shf", sms, clk);
  run<9>("shr", sms, clk);
  run<5>("iadd", sms, clk);
  run<6>("fmul", sms, clk);
  run<7>("fmnmx", sms, clk);
  run<11>("clz+xor", sms, clk);
  run<12>("prmt", sms, clk);
  run<13>("min.u32", sms, clk);
  run<14>("setp+selp", sms, clk);
  run<15>("mad.wide64", sms, clk);
  run<16>("mad.hi+add", sms, clk);
  return 0;
}
