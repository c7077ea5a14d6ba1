// Microbenchmark: streaming u16 reads + pass-1-style scattered int32 stores.
// Models one fold-pass tile = 2187 rows x 256 B (strided by rowlen) -> 16384 outputs.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
#define CK(x) do{cudaError_t e=(x); if(e!=cudaSuccess){printf("err %s line %d\n",cudaGetErrorString(e),__LINE__);return 1;}}while(0)

// mode 0: read only (sum, write 1 value per tile)
// mode 1: read + scattered stores out[slot*ntiles + tile]
// mode 2: read + contiguous stores out[tile*16384 + slot]
template<int MODE>
__global__ void __launch_bounds__(512) tile_kernel(const uint16_t* __restrict__ in, int* __restrict__ out,
    int64_t ntiles, int64_t rowlen_elems, int rows, int cols) {
  // tile t: rows [ (t / C) * rows, +rows ), cols [ (t % C) * cols, +cols )
  const int64_t C = rowlen_elems / cols;
  for (int64_t t = blockIdx.x; t < ntiles; t += gridDim.x) {
    const int64_t aH = t / C, c = t % C;
    const uint16_t* base = in + aH * rows * rowlen_elems + c * cols;
    uint32_t acc = 0;
    const int chunks = cols / 8;   // 16B chunks per row
    for (int i = threadIdx.x; i < rows * chunks; i += blockDim.x) {
      int r = i / chunks, k = i % chunks;
      uint4 v = __ldcs(reinterpret_cast<const uint4*>(base + r * rowlen_elems) + k);
      acc += v.x ^ v.y ^ v.z ^ v.w;
    }
    if (MODE == 0) { if (acc == 0x12345) out[t] = acc; }
    else {
      for (int s = threadIdx.x; s < 16384; s += blockDim.x) {
        int v = acc + s;
        if (MODE == 1) out[(int64_t)s * ntiles + t] = v;
        else out[t * 16384 + s] = v;
      }
    }
  }
}

__global__ void copy_kernel(const uint4* __restrict__ a, uint4* __restrict__ b, int64_t n) {
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) b[i] = a[i];
}
__global__ void read_kernel(const uint4* __restrict__ a, int* out, int64_t n) {
  uint32_t acc = 0;
  for (int64_t i = blockIdx.x * (int64_t)blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) { uint4 v = __ldcs(a + i); acc += v.x ^ v.y ^ v.z ^ v.w; }
  if (acc == 0x1234567) out[0] = acc;
}

int main() {
  const int n = 12;  // n=12: rows 3^12, cols 4096
  const int64_t R = 531441, D = 4096;
  const int Q = 7; const int rows = 2187, cols = 128;
  uint16_t* in; int* out; 
  size_t inb = R * D * 2;
  CK(cudaMalloc(&in, inb)); CK(cudaMemset(in, 1, inb));
  int64_t ntiles = (R / rows) * (D / cols);
  size_t outb = ntiles * 16384 * 4;
  CK(cudaMalloc(&out, outb + (1<<20)));
  printf("in %.2f GB, tiles %ld, out %.2f GB\n", inb/1e9, ntiles, outb/1e9);
  cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
  float ms;
  int sm = 148;
  for (int rep = 0; rep < 2; ++rep) {
  for (int bpsm : {1, 2, 4, 8}) {
    cudaEventRecord(e0); for (int i=0;i<5;++i) read_kernel<<<sm*bpsm, 512>>>((const uint4*)in, out, inb/16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("read_kernel bpsm=%d: %.1f GB/s\n", bpsm, 5*inb/ms/1e6);
  }
  cudaEventRecord(e0); for (int i=0;i<5;++i) copy_kernel<<<sm*4, 512>>>((const uint4*)in, (uint4*)out, outb/16); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
  cudaEventElapsedTime(&ms, e0, e1); printf("copy %.2f GB: %.1f GB/s (r+w)\n", outb/1e9, 5*2*outb/ms/1e6);
  for (int bpsm : {1, 2, 4}) {
    int grid = sm * bpsm;
    cudaEventRecord(e0); for (int i=0;i<5;++i) tile_kernel<0><<<grid, 512>>>(in, out, ntiles, D, rows, cols); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("tile read-only bpsm=%d: %.1f GB/s\n", bpsm, 5*inb/ms/1e6);
    cudaEventRecord(e0); for (int i=0;i<5;++i) tile_kernel<1><<<grid, 512>>>(in, out, ntiles, D, rows, cols); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("tile scattered-store bpsm=%d: %.3f ms  in-GB/s %.1f  (r+w %.1f)\n", bpsm, ms/5, 5*inb/ms/1e6, 5*(inb+outb)/ms/1e6);
    cudaEventRecord(e0); for (int i=0;i<5;++i) tile_kernel<2><<<grid, 512>>>(in, out, ntiles, D, rows, cols); cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
    cudaEventElapsedTime(&ms, e0, e1); printf("tile contiguous-store bpsm=%d: %.3f ms  in-GB/s %.1f  (r+w %.1f)\n", bpsm, ms/5, 5*inb/ms/1e6, 5*(inb+outb)/ms/1e6);
  }
  }
  return 0;
}
