// Micro-benchmark: tcgen05.mma (kind::f16, M=128, K=16) with the A operand in
// TMEM ("TS") vs shared memory ("SS"), and the cost of staging A into TMEM
// with tcgen05.cp (smem -> TMEM, 128x256b = one 128x16 bf16 tile).
// One CTA per SM, operands resident (contents irrelevant).
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2502_11618_b200/csrc mma_ts_rate.cu
#include <stdio.h>

#include "umma.cuh"

using namespace ls::umma;

__device__ __forceinline__ void mma_ts(uint32_t d_tmem, uint32_t a_tmem, uint64_t bdesc,
                                       uint32_t idesc, uint32_t accumulate) {
    asm volatile(
        "{\n\t"
        ".reg .pred p;\n\t"
        "setp.ne.b32 p, %4, 0;\n\t"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], [%1], %2, %3, p;\n\t"
        "}" ::"r"(d_tmem),
        "r"(a_tmem), "l"(bdesc), "r"(idesc), "r"(accumulate)
        : "memory");
}

__device__ __forceinline__ void tmem_cp(uint32_t taddr, uint64_t sdesc) {
    asm volatile("tcgen05.cp.cta_group::1.128x256b [%0], %1;" ::"r"(taddr), "l"(sdesc) : "memory");
}

// MODE 0: SS.  MODE 1: TS (A tiles already in TMEM).  MODE 2: TS with one
// tcgen05.cp of a fresh A tile every REUSE MMAs.
template <int N, int MODE, int REUSE>
__global__ void k_rate(int iters, long long *cycles) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
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
        const uint64_t ad = smem_desc(smem_u32(smem), 64, kSwizzle64B);
        const uint64_t bd = smem_desc(smem_u32(smem) + 32768, 64, kSwizzle64B);
        const uint64_t cpd = smem_desc(smem_u32(smem), 32, kSwizzle32B);
        const uint32_t id = idesc_bf16(128, N);
        const uint32_t a_base = tmem + 256;  // A tiles at columns 256.. (8 columns each)
        long long t0 = clock64();
        for (int i = 0; i < iters; ++i) {
            if (MODE == 0) {
                mma_bf16(tmem, ad + 2 * (i & 3), bd, id, 1u);
            } else if (MODE == 1) {
                mma_ts(tmem, a_base + 8 * (i & 7), bd, id, 1u);
            } else {
                if (i % REUSE == 0) tmem_cp(a_base + 8 * ((i / REUSE) & 7), cpd + 2 * (i & 3));
                mma_ts(tmem, a_base + 8 * ((i / REUSE) & 7), bd, id, 1u);
            }
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

template <int N, int MODE, int REUSE>
void run(long long *d, int n_sm) {
    const int iters = 4096;
    cudaFuncSetAttribute(k_rate<N, MODE, REUSE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         70000);
    k_rate<N, MODE, REUSE><<<n_sm, 128, 70000>>>(iters, d);
    long long h[256];
    cudaMemcpy(h, d, n_sm * sizeof(long long), cudaMemcpyDeviceToHost);
    double avg = 0;
    for (int i = 0; i < n_sm; ++i) avg += h[i];
    avg /= n_sm;
    const double per = avg / iters;
    const double flop_clk = 2.0 * 128 * N * 16 / per;
    printf("N=%3d %s reuse=%d : %6.1f cycles/MMA  %7.0f FLOP/clk/SM (%.0f%% of 8192)\n", N,
           MODE == 0 ? "SS   " : (MODE == 1 ? "TS   " : "TS+cp"), REUSE, per, flop_clk,
           100.0 * flop_clk / 8192.0);
}

int main() {
    long long *d;
    cudaMalloc(&d, 256 * sizeof(long long));
    int n_sm = 148;
    cudaDeviceGetAttribute(&n_sm, cudaDevAttrMultiProcessorCount, 0);
    run<32, 0, 1>(d, n_sm);
    run<32, 1, 1>(d, n_sm);
    run<64, 0, 1>(d, n_sm);
    run<64, 1, 1>(d, n_sm);
    run<96, 0, 1>(d, n_sm);
    run<96, 1, 1>(d, n_sm);
    run<128, 0, 1>(d, n_sm);
    run<128, 1, 1>(d, n_sm);
    run<256, 0, 1>(d, n_sm);
    run<256, 1, 1>(d, n_sm);
    run<32, 2, 1>(d, n_sm);
    run<32, 2, 3>(d, n_sm);
    run<96, 2, 1>(d, n_sm);
    run<96, 2, 3>(d, n_sm);
    run<64, 2, 3>(d, n_sm);
    cudaError_t e = cudaDeviceSynchronize();
    printf("%s\n", cudaGetErrorString(e));
    return 0;
}
