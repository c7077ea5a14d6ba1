// Microbenchmark: the step-(ii) write pattern.  mu (2^14 x 2^14 complex128,
// 4.3 GB) filled XOR-diagonal by XOR-diagonal: a work unit is an aligned block
// of SEG consecutive masks, and every row r of the unit gets one SEG x 16 B
// segment at columns ((r ^ m0) & ~(SEG-1)).  Answers: how fast can the
// assembly's stores go as a function of the segment length and of how many
// CTAs per SM issue them (no transform, values are cheap arithmetic)?
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ void st256(double2 *dst, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// SEG masks per unit; SPLIT CTAs share a unit (each writes rows r with (r >> 13) == part... low-order split)
// BLOCK: part p writes the row block [p d/SPLIT, (p+1) d/SPLIT) (else rows p, p+SPLIT, ...);
// DESYNC: every CTA starts at a different row (CTAs of a real kernel are not in lockstep)
template <int SEG, int SPLIT, bool BLOCK = false, bool DESYNC = false>
__global__ void __launch_bounds__(512) xor_write(double2 *mu, int logd) {
  const int64_t d = (int64_t)1 << logd;
  const int64_t units = (d / SEG) * SPLIT;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int part = (int)(u % SPLIT);
    const int64_t m0 = (u / SPLIT) * SEG;
    const int64_t rows = d / SPLIT;
    const int64_t rot = DESYNC ? ((int64_t)blockIdx.x * 1536) % rows : 0;
    for (int64_t i0 = threadIdx.x; i0 < rows; i0 += blockDim.x) {
      const int64_t i = (i0 + rot) & (rows - 1);
      const int64_t r = BLOCK ? part * rows + i : i * SPLIT + part;
      const int64_t c0 = (r ^ m0) & ~(int64_t)(SEG - 1);
      double2 *dst = mu + r * d + c0;
      const double v = (double)(r + m0);
      if constexpr (SEG == 1) {
        __stcs(dst, make_double2(v, -v));
      } else {
#pragma unroll
        for (int k = 0; k < SEG / 2; ++k) st256(dst + 2 * k, v, -v, v + 1, -v - 1);
      }
    }
  }
}

// Grouped: a CTA (or a CTA pair for SPLIT = 2) writes the G consecutive units of one
// 128-byte line group back to back, rows rotated per group (groups desynchronised).
template <int SEG, int SPLIT, int G>
__global__ void __launch_bounds__(512) xor_write_grouped(double2 *mu, int logd) {
  const int64_t d = (int64_t)1 << logd;
  const int64_t groups = d / (SEG * G);
  const int part = blockIdx.x % SPLIT;
  const int64_t slots = gridDim.x / SPLIT;
  for (int64_t g = blockIdx.x / SPLIT; g < groups; g += slots) {
    const int64_t rows = d / SPLIT;
    const int64_t rot = (g * 1536) % rows;
    for (int k = 0; k < G; ++k) {
      const int64_t m0 = (g * G + k) * SEG;
      for (int64_t i0 = threadIdx.x; i0 < rows; i0 += blockDim.x) {
        const int64_t i = (i0 + rot) & (rows - 1);
        const int64_t r = part * rows + i;
        const int64_t c0 = (r ^ m0) & ~(int64_t)(SEG - 1);
        double2 *dst = mu + r * d + c0;
        const double v = (double)(r + m0);
        if constexpr (SEG == 1) {
          __stcs(dst, make_double2(v, -v));
        } else {
#pragma unroll
          for (int q = 0; q < SEG / 2; ++q) st256(dst + 2 * q, v, -v, v + 1, -v - 1);
        }
      }
    }
  }
}

template <int SEG, int SPLIT, int G>
int rung(double2 *mu, int logd, int bpsm, const char *name) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * bpsm;
  xor_write_grouped<SEG, SPLIT, G><<<grid, 512>>>(mu, logd);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int i = 0; i < 3; ++i) xor_write_grouped<SEG, SPLIT, G><<<grid, 512>>>(mu, logd);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 16.0 * (double)(1LL << (2 * logd));
  printf("%-34s bpsm=%d  %.3f ms  %.1f GB/s\n", name, bpsm, ms / 3, 3 * bytes / ms / 1e6);
  return 0;
}

__global__ void row_write(double4 *mu, int64_t n4) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x)
    st256((double2 *)(mu + i), 1.0, 2.0, 3.0, (double)i);
}

__global__ void read_kernel(const double4 *a, double *out, int64_t n4) {
  double acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n4; i += (int64_t)gridDim.x * blockDim.x) {
    double x, y, z, w;
    asm volatile("ld.global.nc.v4.f64 {%0, %1, %2, %3}, [%4];" : "=d"(x), "=d"(y), "=d"(z), "=d"(w) : "l"(a + i));
    acc += x + y + z + w;
  }
  if (acc == 1234.5) out[0] = acc;
}

template <int SEG, int SPLIT, bool BLOCK = false, bool DESYNC = false>
int run(double2 *mu, int logd, int bpsm, const char *name) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  const int grid = 148 * bpsm;
  xor_write<SEG, SPLIT, BLOCK, DESYNC><<<grid, 512>>>(mu, logd);
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int i = 0; i < 3; ++i) xor_write<SEG, SPLIT, BLOCK, DESYNC><<<grid, 512>>>(mu, logd);
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double bytes = 16.0 * (double)(1LL << (2 * logd));
  printf("%-28s bpsm=%d  %.3f ms  %.1f GB/s\n", name, bpsm, ms / 3, 3 * bytes / ms / 1e6);
  return 0;
}

int main() {
  const int logd = 14;
  const int64_t d = 1LL << logd;
  double2 *mu;
  double *out;
  const size_t bytes = 16 * (size_t)d * d;
  CK(cudaMalloc(&mu, bytes));
  CK(cudaMalloc(&out, 64));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  float ms;
  for (int bpsm : {1, 2, 4}) {
    row_write<<<148 * bpsm, 512>>>((double4 *)mu, bytes / 32);
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) row_write<<<148 * bpsm, 512>>>((double4 *)mu, bytes / 32);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s bpsm=%d  %.3f ms  %.1f GB/s\n", "contiguous write", bpsm, ms / 3, 3 * bytes / ms / 1e6);
    read_kernel<<<148 * bpsm, 512>>>((const double4 *)mu, out, bytes / 64);
    cudaEventRecord(e0);
    for (int i = 0; i < 3; ++i) read_kernel<<<148 * bpsm, 512>>>((const double4 *)mu, out, bytes / 64);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1);
    printf("%-28s bpsm=%d  %.3f ms  %.1f GB/s\n", "contiguous read (half)", bpsm, ms / 3, 3 * bytes / 2 / ms / 1e6);
  }
  for (int bpsm : {1, 2}) {
    run<2, 1, false, true>(mu, logd, bpsm, "seg 32B desync");
    rung<2, 1, 4>(mu, logd, bpsm, "seg 32B grouped 4");
    rung<2, 2, 4>(mu, logd, bpsm, "seg 32B block-split 2 grouped 4");
    rung<1, 1, 8>(mu, logd, bpsm, "seg 16B grouped 8");
    rung<1, 2, 8>(mu, logd, bpsm, "seg 16B block-split 2 grouped 8");
    run<4, 1, false, true>(mu, logd, bpsm, "seg 64B desync");
    rung<4, 1, 2>(mu, logd, bpsm, "seg 64B grouped 2");
    rung<4, 2, 2>(mu, logd, bpsm, "seg 64B block-split 2 grouped 2");
    run<8, 1, false, true>(mu, logd, bpsm, "seg 128B desync");
    rung<8, 8, 1>(mu, logd, bpsm, "seg 128B block-split 8");
  }
  return 0;
}
