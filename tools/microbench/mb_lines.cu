// Microbenchmark: is the assembly's write phase bound per SM or by HBM?
// mu (2^14 x 2^14 complex128, 4.3 GB) written as XOR-diagonal row segments
// (an aligned block of SEG masks gives every row one SEG x 16 B segment at
// columns (r ^ m0) & ~(SEG-1)), rows desynchronised per CTA.  Variants:
//   * st.global.cs.v4.f64 from registers, grid = NSM CTAs (1 per SM) for
//     NSM = 30 .. 148: the per-SM store rate as a function of the SMs writing;
//   * segment length 128 B .. 1 KB;
//   * cp.async.bulk (TMA engine) global <- shared, one bulk op per segment.
// Build: nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o mb_lines mb_lines.cu
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

__device__ __forceinline__ void st256(double2 *dst, double a, double b, double c, double d) {
  asm volatile("st.global.cs.v4.f64 [%0], {%1, %2, %3, %4};" ::"l"(dst), "d"(a), "d"(b), "d"(c), "d"(d) : "memory");
}

// SEG masks per unit, 4 lanes per 128-byte line (as the assembly's write phase)
template <int SEG>
__global__ void __launch_bounds__(512) xor_st(double2 *mu, int logd) {
  const int64_t d = (int64_t)1 << logd;
  const int64_t units = d / SEG;
  const int lane = threadIdx.x & 3;  // 32-byte slot pair within a 128-byte line
  const int tl = threadIdx.x >> 2;
  const int nt = blockDim.x >> 2;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t m0 = u * SEG;
    const int64_t rot = ((int64_t)blockIdx.x * 1536) % d;
    for (int64_t i0 = tl; i0 < d * (SEG / 8); i0 += nt) {
      const int64_t i = ((i0 / (SEG / 8)) + rot) & (d - 1);
      const int seg8 = (int)(i0 % (SEG / 8));
      const int64_t r = i;
      const int64_t c0 = ((r ^ m0) & ~(int64_t)(SEG - 1)) + 8 * seg8 + 2 * lane;
      const double v = (double)(r + m0);
      st256(mu + r * d + c0, v, -v, v + 1, -v - 1);
    }
  }
}

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

// one cp.async.bulk per SEG x 16 B segment, issued by every thread for its rows
template <int SEG, int WAIT>
__global__ void __launch_bounds__(512) xor_bulk(double2 *mu, int logd) {
  __shared__ __align__(128) double2 stage[64 * 8];
  const int64_t d = (int64_t)1 << logd;
  const int64_t units = d / SEG;
  for (int i = threadIdx.x; i < 64 * 8; i += blockDim.x) stage[i] = make_double2(i, -i);
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  __syncthreads();
  const uint32_t src = smem_u32(stage + 8 * (threadIdx.x & 63));
  int pending = 0;
  for (int64_t u = blockIdx.x; u < units; u += gridDim.x) {
    const int64_t m0 = u * SEG;
    const int64_t rot = ((int64_t)blockIdx.x * 1536) % d;
    for (int64_t i0 = threadIdx.x; i0 < d; i0 += blockDim.x) {
      const int64_t r = (i0 + rot) & (d - 1);
      const int64_t c0 = (r ^ m0) & ~(int64_t)(SEG - 1);
      double2 *dst = mu + r * d + c0;
#pragma unroll
      for (int k = 0; k < SEG / 8; ++k)
        asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], 128;" ::"l"(dst + 8 * k), "r"(src)
                     : "memory");
      asm volatile("cp.async.bulk.commit_group;" ::: "memory");
      if (++pending >= WAIT) {
        asm volatile("cp.async.bulk.wait_group.read %0;" ::"n"(WAIT / 2) : "memory");
        pending = WAIT / 2;
      }
    }
  }
  asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
}

template <typename K>
int timeit(K launch, const char *name, int nsm, int64_t bytes) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  launch();
  CK(cudaDeviceSynchronize());
  cudaEventRecord(e0);
  for (int i = 0; i < 3; ++i) launch();
  cudaEventRecord(e1);
  CK(cudaEventSynchronize(e1));
  float ms;
  cudaEventElapsedTime(&ms, e0, e1);
  const double gbs = 3.0 * (double)bytes / ms / 1e6;
  printf("%-34s ctas=%3d  %.3f ms  %7.1f GB/s  %5.1f GB/s per CTA\n", name, nsm, ms / 3, gbs, gbs / nsm);
  return 0;
}

int main() {
  const int logd = 14;
  const int64_t d = 1LL << logd;
  double2 *mu;
  const int64_t bytes = 16 * d * d;
  CK(cudaMalloc(&mu, bytes));
  for (int nsm : {30, 60, 90, 120, 148}) {
    timeit([&] { xor_st<8><<<nsm, 512>>>(mu, logd); }, "st.v4 seg 128B", nsm, bytes);
    timeit([&] { xor_bulk<8, 16><<<nsm, 512>>>(mu, logd); }, "bulk seg 128B", nsm, bytes);
  }
  for (int bpsm : {1, 2}) {
    const int g = 148 * bpsm;
    timeit([&] { xor_st<16><<<g, 512>>>(mu, logd); }, "st.v4 seg 256B", g, bytes);
    timeit([&] { xor_st<32><<<g, 512>>>(mu, logd); }, "st.v4 seg 512B", g, bytes);
    timeit([&] { xor_st<64><<<g, 512>>>(mu, logd); }, "st.v4 seg 1KB", g, bytes);
    timeit([&] { xor_bulk<16, 16><<<g, 512>>>(mu, logd); }, "bulk seg 256B", g, bytes);
    timeit([&] { xor_bulk<8, 4><<<g, 512>>>(mu, logd); }, "bulk seg 128B wait4", g, bytes);
    timeit([&] { xor_bulk<8, 64><<<g, 512>>>(mu, logd); }, "bulk seg 128B wait64", g, bytes);
  }
  return 0;
}
