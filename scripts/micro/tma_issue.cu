// Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o scripts/micro/tma_issue scripts/micro/tma_issue.cu
// Microbenchmark: cost of issuing 1-D bulk copies (cp.async.bulk) from one thread, and the
// copy completion time, per SM, with all 148 SMs loading from HBM at once.
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>
__device__ __forceinline__ uint32_t su(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }
__global__ void k(const char *src, size_t stride, int bytes, int reps, unsigned long long *out) {
    extern __shared__ __align__(128) char sm[];
    __shared__ uint64_t bar;
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(su(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;");
    }
    __syncthreads();
    if (threadIdx.x != 0) return;
    unsigned long long t_issue = 0, t_total = 0;
    const char *base = src + (size_t)blockIdx.x * stride;
    for (int r = 0; r < reps; ++r) {
        const long long t0 = clock64();
        asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(su(&bar)), "r"(bytes) : "memory");
        const int chunk = 4096;
        for (int o = 0; o < bytes; o += chunk) {
            const int n = bytes - o < chunk ? bytes - o : chunk;
            asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];"
                         ::"r"(su(sm + o)), "l"(base + (size_t)r * bytes + o), "r"(n), "r"(su(&bar)) : "memory");
        }
        const long long t1 = clock64();
        asm volatile("{\n\t.reg .pred p;\n\tW: mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n\t@!p bra W;\n\t}"
                     ::"r"(su(&bar)), "r"(r & 1) : "memory");
        const long long t2 = clock64();
        t_issue += t1 - t0;
        t_total += t2 - t0;
    }
    atomicAdd(out, t_issue);
    atomicAdd(out + 1, t_total);
}
int main() {
    const int sms = 148, reps = 64;
    const size_t stride = (size_t)reps * 64 * 1024;
    char *src;
    cudaMalloc(&src, stride * sms);
    cudaMemset(src, 1, stride * sms);
    unsigned long long *out;
    cudaMalloc(&out, 16);
    cudaFuncSetAttribute(k, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024);
    for (int bytes : {256, 1024, 4096, 6144, 12288, 16384, 32768, 65536}) {
        for (int pass = 0; pass < 2; ++pass) {
            cudaMemset(out, 0, 16);
            k<<<sms, 32, 64 * 1024>>>(src, stride, bytes, reps, out);
            cudaDeviceSynchronize();
        }
        unsigned long long h[2];
        cudaMemcpy(h, out, 16, cudaMemcpyDeviceToHost);
        const double is = (double)h[0] / (sms * reps), tt = (double)h[1] / (sms * reps);
        printf("bytes %6d  issue %8.1f cyc (%.1f B/cyc)  complete %8.1f cyc (%.1f B/cyc/SM)\n", bytes, is,
               bytes / is, tt, bytes / tt);
    }
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
