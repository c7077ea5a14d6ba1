// isolated check of the mbarrier primitives used by tile_tma_kernel
#include <cstdio>
#include <cstdint>
__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ uint32_t try_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.try_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok;
}
__device__ uint32_t test_wait(uint64_t *bar, uint32_t parity) {
    uint32_t ok;
    asm volatile("{\n.reg .pred p;\nmbarrier.test_wait.parity.shared::cta.b64 p, [%1], %2;\nselp.u32 %0, 1, 0, p;\n}\n"
                 : "=r"(ok) : "r"(smem_u32(bar)), "r"(parity) : "memory");
    return ok;
}
__device__ uint64_t st(uint64_t *bar) { uint64_t s; asm volatile("ld.shared.b64 %0, [%1];" : "=l"(s) : "r"(smem_u32(bar))); return s; }
__global__ void k() {
    __shared__ uint64_t bar[2];
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[0])), "r"(8) : "memory");
        asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(&bar[1])), "r"(8) : "memory");
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    if (threadIdx.x == 0) printf("fresh: state %llx test0 %u test1 %u\n", (unsigned long long)st(&bar[0]), test_wait(&bar[0], 0), test_wait(&bar[0], 1));
    __syncthreads();
    if (threadIdx.x < 8) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[0])) : "memory");
    __syncthreads();
    if (threadIdx.x == 0) printf("after 8 arrivals (1 warp): state %llx test0 %u test1 %u\n", (unsigned long long)st(&bar[0]), test_wait(&bar[0], 0), test_wait(&bar[0], 1));
    __syncthreads();
    // arrivals from 8 lanes spread over 4 lanes each of 2 warps
    if ((threadIdx.x & 31) < 4 && threadIdx.x < 64) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&bar[1])) : "memory");
    __syncthreads();
    if (threadIdx.x == 0) printf("bar1 after 8 arrivals (2 warps): state %llx test0 %u test1 %u\n", (unsigned long long)st(&bar[1]), test_wait(&bar[1], 0), test_wait(&bar[1], 1));
    // arrive with an explicit count operand
    __syncthreads();
    if (threadIdx.x < 8) { uint64_t tok; asm volatile("mbarrier.arrive.shared::cta.b64 %0, [%1];" : "=l"(tok) : "r"(smem_u32(&bar[0])) : "memory"); }
    __syncthreads();
    if (threadIdx.x == 0) printf("bar0 after 8 more (token form): state %llx test0 %u test1 %u\n", (unsigned long long)st(&bar[0]), test_wait(&bar[0], 0), test_wait(&bar[0], 1));
}
int main() { k<<<1, 128>>>(); cudaError_t e = cudaDeviceSynchronize(); printf("rc %s\n", cudaGetErrorString(e)); return 0; }
