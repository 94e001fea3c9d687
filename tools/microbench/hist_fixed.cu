// Histogram-update microbenchmark for the fill kernel's interval histograms
// (sm_100a): the shared-memory layout and access pattern of the cfg2/cfg4
// fill ([interval][axis] rows, lane-spread axes, intervals random inside a
// stratum window), one CTA of NT threads per SM, D updates of one w2 per
// "evaluation".  Modes:
//   0  f64 atomicAdd (LDS/DADD/ATOMS.CAST loop) + u32 count   (round-1 fill)
//   1  fixed point: u64 lo atomicAdd (value returned, carry) + u64 hi word
//      [count:24 | sum bits 64..103] atomicAdd                (16 B per bin)
//   2  fixed point: u64 lo atomicAdd (returned) + u32 count + u32 hi only on
//      carry / large values                                      (16 B per bin)
//   3  f64 atomicAdd only (no counts)
//   4  u64 lo atomicAdd without return + u32 count (lower bound of mode 2)
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 hist_fixed.cu -o hf
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("CUDA %s @%d\n",cudaGetErrorString(e),__LINE__); return 1;}}while(0)

template <int MODE, int D, int NT>
__global__ void __launch_bounds__(NT, 1) histk(double *out, int evals, int ng, int win) {
  extern __shared__ __align__(16) unsigned char sm[];
  constexpr int HS = D <= 8 ? 8 : 16;
  const int nb = HS * ng;
  double *hw = (double *)sm;
  unsigned long long *lo = (unsigned long long *)sm;
  unsigned long long *hi = lo + nb;
  unsigned *cnt = (unsigned *)(MODE == 0 || MODE == 3 ? (void *)(hw + nb) : (void *)(lo + nb));
  unsigned *hi32 = cnt + nb;
  for (int i = threadIdx.x; i < 2 * nb; i += NT) lo[i] = 0ull;
  __syncthreads();
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned x = threadIdx.x * 2654435761u + blockIdx.x * 97u + 1;
  // each warp sits in its own stratum window (warps spread over the plan)
  unsigned wbase = (warp * 7919u) % (ng - win);
  double w2 = 1.0 + lane * 1e-3;
  for (int e = 0; e < evals; e++) {
    if ((e & 255) == 0) wbase = (wbase + 104729u * (warp + 1)) % (ng - win);
    int idx[D];
#pragma unroll
    for (int s = 0; s < D; s++) {
      x = x * 1664525u + 1013904223u;
      const int iv = wbase + (x >> 8) % win;
      const int ax = D == 8 ? (s ^ (lane & 7)) : (s + lane) % D;
      idx[s] = iv * HS + ax;
    }
    w2 = w2 * 1.0000001;
    if (MODE == 0 || MODE == 3) {
#pragma unroll
      for (int s = 0; s < D; s++) {
        atomicAdd(&hw[idx[s]], w2);
        if (MODE == 0) atomicAdd(&cnt[idx[s]], 1u);
      }
    } else {
      // w2 * 2^s as a 104-bit integer (hi, lo)
      const double y = w2 * 0x1p70;
      unsigned long long vh = (unsigned long long)(y * 0x1p-64);
      unsigned long long vl = (unsigned long long)(y - (double)vh * 0x1p64);
      if (MODE == 1) {
        unsigned long long old[D];
#pragma unroll
        for (int s = 0; s < D; s++) old[s] = atomicAdd(&lo[idx[s]], vl);
#pragma unroll
        for (int s = 0; s < D; s++) {
          const unsigned long long c = old[s] + vl < old[s] ? 1ull : 0ull;
          atomicAdd(&hi[idx[s]], (1ull << 40) + vh + c);
        }
      } else if (MODE == 2) {
        unsigned long long old[D];
#pragma unroll
        for (int s = 0; s < D; s++) { old[s] = atomicAdd(&lo[idx[s]], vl); atomicAdd(&cnt[idx[s]], 1u); }
#pragma unroll
        for (int s = 0; s < D; s++) {
          const unsigned c = old[s] + vl < old[s] ? 1u : 0u;
          if (c | (unsigned)vh) atomicAdd(&hi32[idx[s]], (unsigned)vh + c);
        }
      } else if (MODE == 4) {
#pragma unroll
        for (int s = 0; s < D; s++) { atomicAdd(&lo[idx[s]], vl); atomicAdd(&cnt[idx[s]], 1u); }
      } else if (MODE == 5) {   // one u32 ATOMS.ADD of a value per update
#pragma unroll
        for (int s = 0; s < D; s++) atomicAdd(&cnt[idx[s]], (unsigned)vl);
      } else if (MODE == 6) {   // one u32 ATOMS.ADD with the old value returned
        unsigned acc = 0;
#pragma unroll
        for (int s = 0; s < D; s++) acc += atomicAdd(&cnt[idx[s]], (unsigned)vl);
        if (acc == 12345u) out[0] = 1.0;
      } else if (MODE == 7) {   // two u32 ADD limbs (no return) + POPC count
#pragma unroll
        for (int s = 0; s < D; s++) {
          atomicAdd(&cnt[idx[s]], 1u);
          atomicAdd(&hi32[idx[s]], (unsigned)vl);
          atomicAdd(&((unsigned *)hi)[idx[s]], (unsigned)(vl >> 32));
        }
      } else if (MODE == 8) {   // POPC count only
#pragma unroll
        for (int s = 0; s < D; s++) atomicAdd(&cnt[idx[s]], 1u);
      } else if (MODE == 10 || MODE == 11) {
        // the fill's fixed-point design: per-bin scale exponent in the count
        // word's top byte (MODE 10: count atomic returns it) or per-axis in a
        // register (MODE 11: POPC count); q = RN(w2 2^k) by one DFMA against
        // 2^52; u32 lo limb with return, hi limb gets q_hi + carry
        unsigned ex[D];
        if (MODE == 10) {
#pragma unroll
          for (int s = 0; s < D; s++) ex[s] = atomicAdd(&cnt[idx[s]], 1u) >> 24;
        } else {
#pragma unroll
          for (int s = 0; s < D; s++) { atomicAdd(&cnt[idx[s]], 1u); ex[s] = (unsigned)s; }
        }
        unsigned ql[D], qh[D];
#pragma unroll
        for (int s = 0; s < D; s++) {
          const double sc = __hiloint2double((int)((1023u + 40u + ex[s]) << 20), 0);
          const double y = __fma_rn(w2, sc, 0x1p52);
          ql[s] = (unsigned)__double2loint(y);
          qh[s] = (unsigned)__double2hiint(y);
        }
        unsigned old[D];
#pragma unroll
        for (int s = 0; s < D; s++) old[s] = atomicAdd(&hi32[idx[s]], ql[s]);
#pragma unroll
        for (int s = 0; s < D; s++) {
          const unsigned c = old[s] + ql[s] < ql[s] ? 1u : 0u;
          atomicAdd(&((unsigned *)hi)[idx[s]], (qh[s] & 0xFFFFFu) + c);
        }
      } else if (MODE == 9) {   // u32 limb with return + carry-conditional second limb + count
        unsigned old[D];
#pragma unroll
        for (int s = 0; s < D; s++) { old[s] = atomicAdd(&hi32[idx[s]], (unsigned)vl); atomicAdd(&cnt[idx[s]], 1u); }
#pragma unroll
        for (int s = 0; s < D; s++) {
          const unsigned c = old[s] + (unsigned)vl < old[s] ? 1u : 0u;
          if (c) atomicAdd(&((unsigned *)hi)[idx[s]], c);
        }
      }
    }
  }
  __syncthreads();
  double acc = 0;
  for (int i = threadIdx.x; i < nb; i += NT) acc += (double)lo[i] + (double)cnt[i];
  out[blockIdx.x * NT + threadIdx.x] = acc;
}

template <int MODE, int D, int NT>
int run(const char *name, int ng, int win, int sms, int clk_khz, double *out) {
  const size_t smem = (size_t)(D <= 8 ? 8 : 16) * ng * 24;
  CK(cudaFuncSetAttribute(histk<MODE, D, NT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  const int evals = 4000;
  histk<MODE, D, NT><<<sms, NT, smem>>>(out, 100, ng, win);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0); cudaEventCreate(&e1);
  cudaEventRecord(e0);
  histk<MODE, D, NT><<<sms, NT, smem>>>(out, evals, ng, win);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms; cudaEventElapsedTime(&ms, e0, e1);
  const double upd = (double)sms * NT * evals * D;
  printf("%-44s d=%d win=%4d NT=%4d: %8.3f ms  %7.3f updates/clk/SM  %6.2f ns/eval/SM-thread-equiv\n", name, D, win, NT, ms,
         upd / (ms * 1e-3) / sms / (clk_khz * 1e3), ms * 1e6 / ((double)evals * NT) );
  return 0;
}

int main() {
  cudaDeviceProp p; CK(cudaGetDeviceProperties(&p, 0));
  int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
  const int sms = p.multiProcessorCount;
  printf("device %s SMs %d clock %d kHz\n", p.name, sms, clk);
  double *out; CK(cudaMalloc(&out, sizeof(double) * sms * 1024));
  for (int rep = 0; rep < 2; rep++) {
    run<0, 8, 768>("f64 CAS + u32 count (round 1)", 1024, 205, sms, clk, out);
    run<1, 8, 768>("fixed: lo(ret) + hi[count|sum] u64", 1024, 205, sms, clk, out);
    run<2, 8, 768>("fixed: lo(ret) + u32 count + hi on carry", 1024, 205, sms, clk, out);
    run<3, 8, 768>("f64 CAS only", 1024, 205, sms, clk, out);
    run<4, 8, 768>("u64 lo (no ret) + u32 count", 1024, 205, sms, clk, out);
    run<0, 6, 1024>("f64 CAS + u32 count (round 1)", 1024, 102, sms, clk, out);
    run<1, 6, 1024>("fixed: lo(ret) + hi[count|sum] u64", 1024, 102, sms, clk, out);
    run<2, 6, 1024>("fixed: lo(ret) + u32 count + hi on carry", 1024, 102, sms, clk, out);
    run<4, 6, 1024>("u64 lo (no ret) + u32 count", 1024, 102, sms, clk, out);
    run<5, 8, 768>("u32 ATOMS.ADD value x1", 1024, 205, sms, clk, out);
    run<6, 8, 768>("u32 ATOMS.ADD value x1 (returned)", 1024, 205, sms, clk, out);
    run<7, 8, 768>("2x u32 ADD limbs + POPC count", 1024, 205, sms, clk, out);
    run<8, 8, 768>("POPC count only", 1024, 205, sms, clk, out);
    run<9, 8, 768>("u32 limb(ret) + carry limb + POPC", 1024, 205, sms, clk, out);
    run<10, 8, 768>("fixed design: cnt(ret,exp) dfma lo(ret) hi", 1024, 205, sms, clk, out);
    run<11, 8, 768>("fixed design: POPC, axis exp, lo(ret) hi", 1024, 205, sms, clk, out);
    run<10, 6, 1024>("fixed design: cnt(ret,exp) dfma lo(ret) hi", 1024, 102, sms, clk, out);
    run<11, 6, 1024>("fixed design: POPC, axis exp, lo(ret) hi", 1024, 102, sms, clk, out);
    run<5, 6, 1024>("u32 ATOMS.ADD value x1", 1024, 102, sms, clk, out);
    run<7, 6, 1024>("2x u32 ADD limbs + POPC count", 1024, 102, sms, clk, out);
    run<8, 6, 1024>("POPC count only", 1024, 102, sms, clk, out);
  }
  return 0;
}
