// Micro-test: does a tcgen05.mma smem descriptor whose start address is NOT
// aligned to the swizzle atom (a 1..7-row shift inside a swizzled K-major
// tile) read the rows the absolute-address swizzle put there?  Tries every
// shift with base_offset 0 and with base_offset = (row shift) pattern phase.
// nvcc -gencode arch=compute_100a,code=sm_100a -O2 -I../paper_2502_11618_b200/csrc umma_shift_test.cu
#include <cuda_bf16.h>
#include <stdio.h>

#include "umma.cuh"

using namespace ls::umma;

template <int ROWB>  // 32, 64 or 128 byte rows (SW32 / SW64 / SW128)
__global__ void k_test(int shift, int base_off_mode, float *out, float *ref, int *bad) {
    extern __shared__ __align__(1024) uint8_t smem_raw[];
    uint8_t *smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
    __shared__ uint64_t bar;
    __shared__ uint32_t tslot;
    constexpr int K = ROWB / 2;      // bf16 per row
    constexpr int ROWS = 160;        // A rows available
    const uint32_t layout = ROWB == 128 ? kSwizzle128B : (ROWB == 64 ? kSwizzle64B : kSwizzle32B);
    // swizzle: XOR 16-byte chunk bits with row-group bits (CUTLASS Swizzle<B,4,3>)
    auto swz = [&](uint32_t a) -> uint32_t {
        const uint32_t bbits = ROWB == 128 ? 3 : (ROWB == 64 ? 2 : 1);
        const uint32_t mask = (1u << bbits) - 1u;
        return a ^ (((a >> 7) & mask) << 4);
    };
    uint8_t *A = smem, *B = smem + 32768;
    for (int i = threadIdx.x; i < ROWS * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        float v = (float)((r * 7 + k * 3) % 17) - 8.0f;
        *reinterpret_cast<__nv_bfloat16 *>(A + swz(r * ROWB + 2 * k)) = __float2bfloat16(v);
    }
    for (int i = threadIdx.x; i < 32 * K; i += blockDim.x) {
        int r = i / K, k = i % K;
        float v = (float)((r * 5 + k * 11) % 13) - 6.0f;
        *reinterpret_cast<__nv_bfloat16 *>(B + swz(r * ROWB + 2 * k)) = __float2bfloat16(v);
    }
    // fence the generic-proxy smem writes before the async proxy (tensor core) reads
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
    if (threadIdx.x < 32) tmem_alloc(&tslot, 32);
    if (threadIdx.x == 0) {
        mbar_init(&bar, 1);
        fence_barrier_init();
    }
    fence_before_sync();
    __syncthreads();
    fence_after_sync();
    const uint32_t tmem = tslot;
    if (threadIdx.x == 0) {
        uint64_t ad = smem_desc(smem_u32(A) + shift * ROWB, ROWB, layout);
        if (base_off_mode) ad |= (uint64_t)(((shift * ROWB) >> 7) & 7) << 49;
        const uint64_t bd = smem_desc(smem_u32(B), ROWB, layout);
        for (int j = 0; j < K / 16; ++j)
            mma_bf16(tmem, ad + 2 * j, bd + 2 * j, idesc_bf16(128, 32), j > 0);
        mma_commit(&bar);
    }
    __syncwarp();
    mbar_wait(&bar, 0);
    fence_after_sync();
    uint32_t r[16];
    const int m = threadIdx.x;  // 128 threads = 4 warps = TMEM lanes
    for (int g = 0; g < 2; ++g) {
        tmem_ld16(tmem + ((uint32_t)((m / 32) * 32) << 16) + g * 16, r);
        for (int i = 0; i < 16; ++i) {
            const int n = g * 16 + i;
            float acc = 0.0f;
            for (int k = 0; k < K; ++k) {
                float a = (float)(((m + shift) * 7 + k * 3) % 17) - 8.0f;
                float b = (float)((n * 5 + k * 11) % 13) - 6.0f;
                acc += a * b;
            }
            out[m * 32 + n] = __uint_as_float(r[i]);
            ref[m * 32 + n] = acc;
            if (fabsf(acc - __uint_as_float(r[i])) > 1e-3f) atomicAdd(bad, 1);
        }
    }
    fence_before_sync();
    __syncthreads();
    if (threadIdx.x < 32) tmem_dealloc(tmem, 32);
}

int main() {
    float *out, *ref;
    int *bad;
    cudaMalloc(&out, 128 * 32 * 4);
    cudaMalloc(&ref, 128 * 32 * 4);
    cudaMalloc(&bad, 4);
    for (int rowb : {32, 64, 128}) {
        for (int mode = 0; mode < 2; ++mode) {
            printf("rowbytes %3d base_offset %s:", rowb, mode ? "phase" : "zero ");
            for (int shift = 0; shift < 9; ++shift) {
                cudaMemset(bad, 0, 4);
                if (rowb == 32) {
                    cudaFuncSetAttribute(k_test<32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
                    k_test<32><<<1, 128, 70000>>>(shift, mode, out, ref, bad);
                } else if (rowb == 64) {
                    cudaFuncSetAttribute(k_test<64>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
                    k_test<64><<<1, 128, 70000>>>(shift, mode, out, ref, bad);
                } else {
                    cudaFuncSetAttribute(k_test<128>, cudaFuncAttributeMaxDynamicSharedMemorySize, 70000);
                    k_test<128><<<1, 128, 70000>>>(shift, mode, out, ref, bad);
                }
                int h = -1;
                cudaError_t e = cudaMemcpy(&h, bad, 4, cudaMemcpyDeviceToHost);
                if (e != cudaSuccess) {
                    printf(" ERR(%s)\n", cudaGetErrorString(e));
                    return 1;
                }
                printf(" s%d:%s", shift, h == 0 ? "ok" : "BAD");
            }
            printf("\n");
        }
    }
    return 0;
}
