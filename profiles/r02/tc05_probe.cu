// Probe of the sm_100a tcgen05 building blocks the join+encode kernel uses:
// TMEM alloc, kind::f16 MMAs from no-swizzle shared-memory descriptors (K-major
// and MN-major operands), commit to an mbarrier, tcgen05.ld of M=128 and M=64
// accumulators.  Runs each candidate (LBO, SBO) assignment and prints which
// ones reproduce the CPU product, and where an M=64 accumulator lands in TMEM.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -o /tmp/tc05_probe profiles/tc05_probe.cu && /tmp/tc05_probe
#include <cuda_fp16.h>
#include <cstdio>
#include <cstdint>
#include <cstdlib>
#include <cmath>

__device__ __forceinline__ uint32_t smem_u32(const void *p) { return (uint32_t)__cvta_generic_to_shared(p); }

__device__ __forceinline__ uint64_t sdesc(uint32_t addr, uint32_t lbo, uint32_t sbo) {
    uint64_t d = 0;
    d |= (uint64_t)((addr >> 4) & 0x3FFF);
    d |= (uint64_t)((lbo >> 4) & 0x3FFF) << 16;
    d |= (uint64_t)((sbo >> 4) & 0x3FFF) << 32;
    d |= (uint64_t)1 << 46;  // version (sm100)
    return d;                // base offset 0, lbo mode 0, SWIZZLE_NONE
}

__host__ __device__ constexpr uint32_t idesc_f16(int M, int N, int amaj, int bmaj) {
    return (1u << 4) | (0u << 7) | (0u << 10) | ((uint32_t)amaj << 15) | ((uint32_t)bmaj << 16) |
           ((uint32_t)(N >> 3) << 17) | ((uint32_t)(M >> 4) << 24);
}

__device__ __forceinline__ void mma_f16(uint32_t dt, uint64_t ad, uint64_t bd, uint32_t id, uint32_t acc) {
    asm volatile(
        "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
        "tcgen05.mma.cta_group::1.kind::f16 [%0], %1, %2, %3, p;\n}\n" ::"r"(dt),
        "l"(ad), "l"(bd), "r"(id), "r"(acc));
}

__device__ __forceinline__ void commit(uint64_t *bar) {
    asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar)));
}

__device__ __forceinline__ void mbar_init(uint64_t *bar, int n) {
    asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;\n" ::"r"(smem_u32(bar)), "r"(n));
}

__device__ __forceinline__ void mbar_wait(uint64_t *bar, uint32_t phase) {
    asm volatile(
        "{\n.reg .pred P1;\nWAIT_%=:\n"
        "mbarrier.try_wait.parity.shared::cta.b64 P1, [%0], %1;\n"
        "@!P1 bra WAIT_%=;\n}\n" ::"r"(smem_u32(bar)),
        "r"(phase));
}

__device__ __forceinline__ void ld16(uint32_t taddr, float (&v)[16]) {
    uint32_t r[16];
    asm volatile(
        "tcgen05.ld.sync.aligned.32x32b.x16.b32 {%0,%1,%2,%3,%4,%5,%6,%7,%8,%9,%10,%11,%12,%13,%14,%15}, [%16];\n"
        : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7]), "=r"(r[8]),
          "=r"(r[9]), "=r"(r[10]), "=r"(r[11]), "=r"(r[12]), "=r"(r[13]), "=r"(r[14]), "=r"(r[15])
        : "r"(taddr));
    asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory");
#pragma unroll
    for (int i = 0; i < 16; ++i) v[i] = __uint_as_float(r[i]);
}

// X: [128 rows][16 k] fp16 stored core-matrix blocked: off(r,k) = (r/8)*256 + (k/8)*128 + (r%8)*16 + (k%8)*2
// W: [64 rows][16 k]  same blocking
// G: [128 k][64 m]    off(k,m) = (k/8)*1024 + (m/8)*128 + (k%8)*16 + (m%8)*2
// out1: [128][64] (X W^T), out2: [128 lanes][16 cols] raw TMEM dump of the M=64 product G^T X
__global__ void probe(const __half *X, const __half *W, const __half *G, float *out1, float *out2, int variant) {
    __shared__ __align__(1024) unsigned char sm[4096 + 2048 + 16384];
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    unsigned char *xs = sm, *ws = sm + 4096, *gs = sm + 6144;
    const int t = threadIdx.x, warp = t >> 5;
    for (int i = t; i < 128 * 16; i += 128) {
        const int r = i / 16, k = i % 16;
        *reinterpret_cast<__half *>(xs + (r / 8) * 256 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) = X[i];
    }
    for (int i = t; i < 64 * 16; i += 128) {
        const int r = i / 16, k = i % 16;
        *reinterpret_cast<__half *>(ws + (r / 8) * 256 + (k / 8) * 128 + (r % 8) * 16 + (k % 8) * 2) = W[i];
    }
    for (int i = t; i < 128 * 64; i += 128) {
        const int k = i / 64, m = i % 64;
        *reinterpret_cast<__half *>(gs + (k / 8) * 1024 + (m / 8) * 128 + (k % 8) * 16 + (m % 8) * 2) = G[i];
    }
    if (warp == 0) {
        asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], 128;\n" ::"r"(smem_u32(&tbase)));
        asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
    }
    if (t == 0) {
        mbar_init(&bar, 1);
        asm volatile("fence.mbarrier_init.release.cluster;\n");
    }
    asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t tb = tbase;
    const uint32_t d1 = tb, d2 = tb + 64;  // columns
    if (t == 0 && !(variant & 8)) {
        // GEMM1 K-major A (X) and B (W): variant bit 0 swaps LBO/SBO
        const uint32_t lbo = (variant & 1) ? 256 : 128, sbo = (variant & 1) ? 128 : 256;
        mma_f16(d1, sdesc(smem_u32(xs), lbo, sbo), sdesc(smem_u32(ws), lbo, sbo), idesc_f16(128, 64, 0, 0), 0);
    }
    if (t == 0 && !(variant & 4)) {
        // GEMM2 M=64 N=16 K=128 in 8 k16 steps; A = G^T MN-major, B = X MN-major (k = row of X)
        // A: m-block stride 128, k-block stride 1024; B: n-block stride 128, k-block stride 256
        // variant bit 1 swaps the LBO/SBO roles for MN-major operands
        for (int ks = 0; ks < 8; ++ks) {
            const uint32_t a_addr = smem_u32(gs) + ks * 2 * 1024;  // 16 k = 2 k-blocks
            const uint32_t b_addr = smem_u32(xs) + ks * 2 * 256;
            uint64_t ad, bd;
            if (variant & 2) {
                ad = sdesc(a_addr, 1024, 128);
                bd = sdesc(b_addr, 256, 128);
            } else {
                ad = sdesc(a_addr, 128, 1024);
                bd = sdesc(b_addr, 128, 256);
            }
            mma_f16(d2, ad, bd, idesc_f16(64, 16, 1, 1), ks > 0);
        }
    }
    if (t == 0) commit(&bar);
    __syncwarp();
    mbar_wait(&bar, 0);
    asm volatile("tcgen05.fence::after_thread_sync;\n");
    const uint32_t lane_base = (uint32_t)(warp * 32) << 16;
    for (int c = 0; c < 64; c += 16) {
        float v[16];
        ld16(d1 + lane_base + c, v);
        for (int i = 0; i < 16; ++i) out1[t * 64 + c + i] = v[i];
    }
    {
        float v[16];
        ld16(d2 + lane_base, v);
        for (int i = 0; i < 16; ++i) out2[t * 16 + i] = v[i];
    }
    asm volatile("tcgen05.fence::before_thread_sync;\n");
    __syncthreads();
    if (warp == 0) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, 128;\n" ::"r"(tb));
}

int main(int argc, char **argv) {
    const int extra = argc > 1 ? atoi(argv[1]) : 0;
    const int nX = 128 * 16, nW = 64 * 16, nG = 128 * 64;
    __half hX[nX], hW[nW], *hG = (__half *)malloc(nG * sizeof(__half));
    float fX[nX], fW[nW], *fG = (float *)malloc(nG * 4);
    srand(1);
    for (int i = 0; i < nX; ++i) { fX[i] = (float)(rand() % 7 - 3); hX[i] = __float2half(fX[i]); }
    for (int i = 0; i < nW; ++i) { fW[i] = (float)(rand() % 9 - 4) * 0.25f; hW[i] = __float2half(fW[i]); }
    for (int i = 0; i < nG; ++i) { fG[i] = (float)(rand() % 5); hG[i] = __float2half(fG[i]); }
    __half *dX, *dW, *dG;
    float *o1, *o2;
    cudaMalloc(&dX, nX * 2); cudaMalloc(&dW, nW * 2); cudaMalloc(&dG, nG * 2);
    cudaMalloc(&o1, 128 * 64 * 4); cudaMalloc(&o2, 128 * 16 * 4);
    cudaMemcpy(dX, hX, nX * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dW, hW, nW * 2, cudaMemcpyHostToDevice);
    cudaMemcpy(dG, hG, nG * 2, cudaMemcpyHostToDevice);
    // references
    static float r1[128 * 64], r2[64 * 16];
    for (int r = 0; r < 128; ++r)
        for (int n = 0; n < 64; ++n) {
            float s = 0; for (int k = 0; k < 16; ++k) s += fX[r * 16 + k] * fW[n * 16 + k];
            r1[r * 64 + n] = s;
        }
    for (int m = 0; m < 64; ++m)
        for (int n = 0; n < 16; ++n) {
            float s = 0; for (int k = 0; k < 128; ++k) s += fG[k * 64 + m] * fX[k * 16 + n];
            r2[m * 16 + n] = s;
        }
    for (int variant = 0; variant < 4; ++variant) {
        cudaMemset(o1, 0, 128 * 64 * 4); cudaMemset(o2, 0, 128 * 16 * 4);
        probe<<<1, 128>>>(dX, dW, dG, o1, o2, variant | extra);
        cudaError_t e = cudaDeviceSynchronize();
        if (e != cudaSuccess) { printf("variant %d: CUDA error %s\n", variant, cudaGetErrorString(e)); return 1; }
        static float h1[128 * 64], h2[128 * 16];
        cudaMemcpy(h1, o1, sizeof h1, cudaMemcpyDeviceToHost);
        cudaMemcpy(h2, o2, sizeof h2, cudaMemcpyDeviceToHost);
        int bad1 = 0;
        for (int i = 0; i < 128 * 64; ++i) bad1 += fabsf(h1[i] - r1[i]) > 1e-3f;
        // locate each reference row m of the M=64 product among the 128 TMEM lanes
        int found = 0;
        printf("variant %d: GEMM1 mismatches %d / %d;  M=64 rows -> lanes:", variant, bad1, 128 * 64);
        for (int m = 0; m < 64; ++m) {
            int lane = -1;
            for (int l = 0; l < 128 && lane < 0; ++l) {
                int ok = 1;
                for (int n = 0; n < 16; ++n) ok &= fabsf(h2[l * 16 + n] - r2[m * 16 + n]) < 1e-2f;
                if (ok) lane = l;
            }
            found += lane >= 0;
            if (m % 8 == 0 || m == 63) printf(" %d->%d", m, lane);
        }
        printf("  (%d/64 rows found)\n", found);
    }
    return 0;
}
