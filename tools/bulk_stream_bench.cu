// bulk_stream_bench.cu -- how fast can one CTA per SM pull a contiguous stream from HBM into a
// shared-memory ring with cp.async.bulk, as a function of the ring's depth and slot size?
// (The window SpMV keeps ~2 ring slots of ~20 KB in flight per SM next to its input windows.)
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/bulk_stream tools/bulk_stream_bench.cu && /tmp/bulk_stream
#include <cstdio>
#include <cstdlib>
#include <algorithm>
#include <cuda_runtime.h>
#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)
__device__ __forceinline__ unsigned smem_u32(const void *p) { return (unsigned)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(unsigned long long *b, unsigned c) { asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(b)), "r"(c) : "memory"); }
__device__ __forceinline__ void mbar_expect_tx(unsigned long long *b, unsigned n) { asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(b)), "r"(n) : "memory"); }
__device__ __forceinline__ void mbar_arrive(unsigned long long *b) { asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(b)) : "memory"); }
template <int HINT>
__device__ __forceinline__ void mbar_wait(unsigned long long *b, unsigned parity) {
    if (HINT > 0)
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1, %2;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity), "r"((unsigned)HINT) : "memory");
    else if (HINT == 0)
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
    else
        asm volatile("{\n.reg .pred p;\nW_%=:\nmbarrier.test_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(smem_u32(b)), "r"(parity) : "memory");
}
__device__ __forceinline__ void bulk_g2s(void *dst, const void *src, unsigned bytes, unsigned long long *bar) {
    asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(smem_u32(dst)), "l"(src), "r"(bytes), "r"(smem_u32(bar)) : "memory");
}
// one producer thread, one consumer warp that reads one word per slot and releases it
template <int HINT>
__global__ void __launch_bounds__(64, 1) stream(const unsigned char *src, size_t per_cta, int slot_bytes, int ns, int pieces,
                                                double *sink) {
    extern __shared__ __align__(128) unsigned char smem[];
    unsigned long long *full = reinterpret_cast<unsigned long long *>(smem + (size_t)ns * slot_bytes);
    unsigned long long *empty = full + ns;
    if (threadIdx.x == 0) {
        for (int s = 0; s < ns; ++s) { mbar_init(&full[s], 1); mbar_init(&empty[s], 1); }
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    __syncthreads();
    const unsigned char *base = src + (size_t)blockIdx.x * per_cta;
    const long long nslots = per_cta / slot_bytes;
    if (threadIdx.x == 32) {
        for (long long q = 0; q < nslots; ++q) {
            const int s = (int)(q % ns);
            if (q >= ns) mbar_wait<HINT>(&empty[s], (unsigned)(((q / ns) - 1) & 1));
            mbar_expect_tx(&full[s], slot_bytes);
            const int pb = slot_bytes / pieces;
            for (int p = 0; p < pieces; ++p) bulk_g2s(smem + (size_t)s * slot_bytes + p * pb, base + q * slot_bytes + p * pb, pb, &full[s]);
        }
    } else if (threadIdx.x < 32) {
        double acc = 0.0;
        for (long long q = 0; q < nslots; ++q) {
            const int s = (int)(q % ns);
            mbar_wait<HINT>(&full[s], (unsigned)((q / ns) & 1));
            acc += reinterpret_cast<const double *>(smem + (size_t)s * slot_bytes)[threadIdx.x];
            __syncwarp();
            if (threadIdx.x == 0) mbar_arrive(&empty[s]);
        }
        if (acc == 1.2345) sink[0] = acc;
    }
}
int main() {
    const size_t total = 888ull << 20;      // ~the window SpMV's per-launch bulk traffic
    unsigned char *d; double *sink;
    CK(cudaMalloc(&d, total + (1 << 20))); CK(cudaMemset(d, 1, total)); CK(cudaMalloc(&sink, 8));
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    CK(cudaFuncSetAttribute(stream<2000>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    CK(cudaFuncSetAttribute(stream<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    CK(cudaFuncSetAttribute(stream<-1>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    CK(cudaFuncSetAttribute(stream<100>, cudaFuncAttributeMaxDynamicSharedMemorySize, 227 * 1024));
    for (int hint : {2000, 100, 0, -1})
    for (int pieces : {1, 4})
    for (int grid : {148}) {
        for (int slot_kb : {8, 16}) {
            for (int ns : {2, 4}) {
                const size_t smem = (size_t)ns * slot_kb * 1024 + 16 * ns;
                if (smem * (grid / 148) > 227 * 1024) continue;
                const size_t per = total / grid / (slot_kb * 1024) * (slot_kb * 1024);
                float best = 1e9;
                for (int rep = 0; rep < 4; ++rep) {
                    cudaEventRecord(e0);
                    if (hint == 2000) stream<2000><<<grid, 64, smem>>>(d, per, slot_kb * 1024, ns, pieces, sink);
                    else if (hint == 100) stream<100><<<grid, 64, smem>>>(d, per, slot_kb * 1024, ns, pieces, sink);
                    else if (hint == 0) stream<0><<<grid, 64, smem>>>(d, per, slot_kb * 1024, ns, pieces, sink);
                    else stream<-1><<<grid, 64, smem>>>(d, per, slot_kb * 1024, ns, pieces, sink);
                    cudaEventRecord(e1); CK(cudaEventSynchronize(e1));
                    float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
                }
                printf("hint %4d pieces %d  grid %3d  slot %2d KB x %d (%3d KB in ring/CTA)  %7.1f us  %5.2f TB/s  %5.1f GB/s per SM\n", hint, pieces, grid, slot_kb, ns,
                       slot_kb * ns, best * 1e3, per * grid / (best * 1e-3) / 1e12, per * grid / (best * 1e-3) / 1e9 / 148);
            }
        }
    }
    return 0;
}
