// Micro-benchmark: cycles per tcgen05.mma (kind::f16, M=128, K=16) issued
// back to back by one thread, as a function of N, the operand swizzle width
// and how many independent accumulators the sequence rotates through.
// One CTA per SM, operands resident in shared memory (contents irrelevant).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2502_11618_b200/csrc mma_rate.cu
#include <stdio.h>

#include "umma.cuh"

using namespace ls::umma;

template <int N, int ROWB, int NACC>
__global__ void k_rate(int iters, long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    const uint32_t layout = ROWB == 128 ? kSwizzle128B : (ROWB == 64 ? kSwizzle64B : kSwizzle32B);
    for (int i = threadIdx.x; i < 64 * 1024 / 4; i += blockDim.x)
        reinterpret_cast<uint32_t *>(smem)[i] = 0x3c003c00u;
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) tmem_alloc(&tslot, 512);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        const uint64_t ad = smem_desc(smem_u32(smem), ROWB, layout);
        const uint64_t bd = smem_desc(smem_u32(smem) + 32768, ROWB, layout);
        const uint32_t id = idesc_bf16(128, N);
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
#pragma unroll
            for (int a = 0; a < NACC; ++a)
                mma_bf16(tmem + a * N, ad + 2 * (a & 3), bd, id, 1u);
        }
        mma_commit(&bar);
        mbar_wait(&bar, 0);
        long long t1 = clock64();
        cycles[blockIdx.x] = t1 - t0;
    }
    fence_before_sync();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 512);
}

template <int N, int ROWB, int NACC>
void run(long long *d, int n_sm) {
    const int iters = 4096 / NACC;
    cudaFuncSetAttribute(k_rate<N, ROWB, NACC>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
    k_rate<N, ROWB, NACC><<<n_sm, 128, 70000>>>(iters, d);
    long long h[256];
    cudaMemcpy(h, d, n_sm * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < n_sm; ++i) avg += h[i];
    avg /= n_sm;
    const double per = avg / (iters * NACC);
    const double flop_clk = 2.0 * 128 * N * 16 / per;
    printf("N=%3d rowB=%3d acc=%d : %6.1f cycles/MMA  %7.0f FLOP/clk/SM\n", N, ROWB, NACC, per,
           flop_clk);
}

int main() {
    long long *d;
    cudaMalloc(&d, 256 * sizeof(long long));
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
    run<96, 64, 1>(d, n_sm);
    run<96, 32, 1>(d, n_sm);
    run<80, 64, 1>(d, n_sm);
    run<112, 64, 1>(d, n_sm);
    run<32, 64, 1>(d, n_sm);
    run<32, 64, 4>(d, n_sm);
    run<32, 32, 4>(d, n_sm);
    run<32, 128, 4>(d, n_sm);
    run<64, 64, 1>(d, n_sm);
    run<64, 64, 4>(d, n_sm);
    run<64, 128, 4>(d, n_sm);
    run<128, 128, 1>(d, n_sm);
    run<128, 128, 2>(d, n_sm);
    run<256, 128, 1>(d, n_sm);
    run<256, 128, 2>(d, n_sm);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
