// Microbenchmark 2: pass-1 output write patterns.
// Each "tile" reads 2187 rows x 256 B (u16, strided by rowlen) and writes 64 KB of int32 results.
// Layout A (scattered, run L bytes): the tile's 16384 words are grouped in runs of L/4 words;
//   run j of tile t goes to out[(j * ntiles + t) * (L/4) ...]  (W = L/4 adjacent tiles share a 4W-byte... no:
//   here each tile owns its run, runs of different tiles interleave) -> models W-adjacent-tile coalescing.
// Layout L2S: write the tile contiguously into a per-CTA scratch ring of W tiles, then after W tiles
//   re-read the ring and write runs of 4W bytes (true transposition through L2).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

template <int RUNW>  // words per run
__global__ void __launch_bounds__(512) runs_kernel(const uint16_t* __restrict__ in, int* __restrict__ out,
    int64_t ntiles, int64_t rowlen_elems, int rows, int cols) {
  const int64_t C = rowlen_elems / cols;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t aH = t / C, c = t % C;
    const uint16_t* base = in + aH * rows * rowlen_elems + c * cols;
    uint32_t acc = 0;
    const int chunks = cols / 8;
    for (int i = threadIdx.x; i < rows * chunks; i += blockDim.x) {
      int r = i / chunks, k = i % chunks;
      uint4 v = __ldcs(reinterpret_cast<const uint4*>(base + r * rowlen_elems) + k);
      acc += v.x ^ v.y ^ v.z ^ v.w;
    }
    const int nruns = 16384 / RUNW;
    for (int j = threadIdx.x; j < nruns; j += blockDim.x) {
      int* dst = out + ((int64_t)j * ntiles + t) * RUNW;
      if constexpr (RUNW == 1) dst[0] = acc + j;
      else if constexpr (RUNW == 2) *reinterpret_cast<int2*>(dst) = make_int2(acc, j);
      else {
#pragma unroll
        for (int q = 0; q < RUNW; q += 4) *reinterpret_cast<int4*>(dst + q) = make_int4(acc, j, q, 1);
      }
    }
  }
}

// L2-scratch transpose: W consecutive tiles per CTA batch
template <int W>
__global__ void __launch_bounds__(512) l2s_kernel(const uint16_t* __restrict__ in, int* __restrict__ out,
    int* __restrict__ scratch, int64_t ntiles, int64_t rowlen_elems, int rows, int cols) {
  const int64_t C = rowlen_elems / cols;
  int* my = scratch + (int64_t)blockIdx.x * W * 16384;
  for (int64_t tb = (int64_t)blockIdx.x * W; tb < ntiles; tb += (int64_t)gridDim.x * W) {
    for (int w = 0; w < W; ++w) {
      const int64_t t = tb + w;
      const int64_t aH = t / C, c = t % C;
      const uint16_t* base = in + aH * rows * rowlen_elems + c * cols;
      uint32_t acc = 0;
      const int chunks = cols / 8;
      for (int i = threadIdx.x; i < rows * chunks; i += blockDim.x) {
        int r = i / chunks, k = i % chunks;
        uint4 v = __ldcs(reinterpret_cast<const uint4*>(base + r * rowlen_elems) + k);
        acc += v.x ^ v.y ^ v.z ^ v.w;
      }
      for (int s = threadIdx.x * 4; s < 16384; s += blockDim.x * 4)
        *reinterpret_cast<int4*>(my + w * 16384 + s) = make_int4(acc, s, w, 1);
    }
    __syncthreads();
    // transpose: slot s, W words from the W tiles -> out[s * ntiles + tb .. +W)
    for (int s = threadIdx.x; s < 16384; s += blockDim.x) {
      int v[W];
#pragma unroll
      for (int w = 0; w < W; ++w) v[w] = my[w * 16384 + s];
      int* dst = out + (int64_t)s * ntiles + tb;
#pragma unroll
      for (int q = 0; q < W; q += 4) *reinterpret_cast<int4*>(dst + q) = make_int4(v[q], v[q + 1], v[q + 2], v[q + 3]);
    }
    __syncthreads();
  }
}

int main() {
  const int64_t R = 531441, D = 4096;
  const int rows = 2187, cols = 128;
  uint16_t* in; int* out; int* scratch;
  size_t inb = R * D * 2;
  CK(cudaMalloc(&in, inb)); CK(cudaMemset(in, 1, inb));
  int64_t ntiles = (R / rows) * (D / cols);
  size_t outb = ntiles * 16384 * 4;
  CK(cudaMalloc(&out, outb + (1<<20)));
  CK(cudaMalloc(&scratch, (size_t)148 * 4 * 16 * 16384 * 4));
  printf("in %.2f GB, tiles %ld, out %.2f GB\n", inb/1e9, ntiles, outb/1e9);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  auto rep = [&](const char* name, auto launch) {
    launch(); cudaEventRecord(e0); for (int i=0;i<5;++i) launch(); cudaEventRecord(e1); cudaEventSynchronize(e1);
    cudaEventElapsedTime(&ms, e0, e1); ms /= 5;
    printf("%-28s %.3f ms  in-GB/s %.1f  (r+w %.1f)\n", name, ms, inb/ms/1e6, (inb+outb)/ms/1e6);
  };
  for (int bpsm : {2, 4}) {
    int g = 148 * bpsm;
    printf("-- blocks/SM %d\n", bpsm);
    rep("run 4B", [&]{ runs_kernel<1><<<g,512>>>(in,out,ntiles,D,rows,cols); });
    rep("run 8B", [&]{ runs_kernel<2><<<g,512>>>(in,out,ntiles,D,rows,cols); });
    rep("run 16B", [&]{ runs_kernel<4><<<g,512>>>(in,out,ntiles,D,rows,cols); });
    rep("run 32B", [&]{ runs_kernel<8><<<g,512>>>(in,out,ntiles,D,rows,cols); });
    rep("run 64B", [&]{ runs_kernel<16><<<g,512>>>(in,out,ntiles,D,rows,cols); });
    rep("run 128B", [&]{ runs_kernel<32><<<g,512>>>(in,out,ntiles,D,rows,cols); });
  }
  for (int bpsm : {1, 2}) {
    int g = 148 * bpsm;
    printf("-- L2 scratch, blocks/SM %d\n", bpsm);
    rep("l2s W=4", [&]{ l2s_kernel<4><<<g,512>>>(in,out,scratch,ntiles,D,rows,cols); });
    rep("l2s W=8", [&]{ l2s_kernel<8><<<g,512>>>(in,out,scratch,ntiles,D,rows,cols); });
  }
  CK(cudaGetLastError());
  return 0;
}
