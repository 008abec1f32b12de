// gather_bench.cu -- ceiling of the random 8-byte gather that bounds config 5's
// SpMV (random +-50000 band, 22.7 nonzeros per row, n = 2,000,000).
//
//   nvcc -O3 -gencode arch=compute_100a,code=sm_100a -o /tmp/gather_bench tools/gather_bench.cu
//   /tmp/gather_bench
//
// Each kernel streams an int32 column list (coalesced) and sums x[col] per
// thread (no smem, no ordering constraint): the pure cost of the gathers.
// Column lists: (a) config 5's CSR order (random within +-50000 of the row),
// (b) the same sorted by column inside blocks of R rows, (c) a sequential
// baseline.  Also varies the load path (ld.global.nc vs ld.global.cg).
#include <cstdio>
#include <cstdlib>
#include <vector>
#include <algorithm>
#include <random>
#include <cuda_runtime.h>

template <int PER, bool NC>
__global__ void gather(const int *__restrict__ col, long long nnz, const double *__restrict__ x, double *out) {
    const long long tid = blockIdx.x * (long long)blockDim.x + threadIdx.x;
    const long long nth = (long long)gridDim.x * blockDim.x;
    double acc = 0.0;
    for (long long k = tid; k < nnz; k += nth * PER) {
        int c[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) c[j] = (k + j * nth < nnz) ? __ldcs(col + k + j * nth) : 0;
        double v[PER];
#pragma unroll
        for (int j = 0; j < PER; ++j) v[j] = NC ? __ldg(x + c[j]) : __ldcg(x + c[j]);
#pragma unroll
        for (int j = 0; j < PER; ++j) acc += v[j];
    }
    if (acc == 12345.678) out[0] = acc;   // keep the loads alive
}

int main() {
    const long long n = 2000000, per_row = 23, band = 50000;
    const long long nnz = n * per_row;
    std::mt19937_64 rng(1);
    std::vector<int> csr(nnz);
    for (long long r = 0; r < n; ++r)
        for (long long j = 0; j < per_row; ++j) {
            long long c = r + (long long)(rng() % (2 * band + 1)) - band;
            csr[r * per_row + j] = (int)std::min(std::max(c, 0LL), n - 1);
        }
    for (long long r = 0; r < n; ++r) std::sort(csr.begin() + r * per_row, csr.begin() + (r + 1) * per_row);
    auto blocked = [&](long long R) {
        std::vector<int> v = csr;
        for (long long b = 0; b < n; b += R)
            std::sort(v.begin() + b * per_row, v.begin() + std::min(n, b + R) * per_row);
        return v;
    };
    std::vector<int> seq(nnz);
    for (long long k = 0; k < nnz; ++k) seq[k] = (int)(k % n);
    struct Case { const char *name; std::vector<int> v; };
    std::vector<Case> cases = {{"csr-order", csr}, {"sorted R=1024", blocked(1024)},
                               {"sorted R=8192", blocked(8192)}, {"sorted R=65536", blocked(65536)},
                               {"sequential", seq}};
    int *dcol; double *dx, *dout;
    cudaMalloc(&dcol, nnz * 4); cudaMalloc(&dx, n * 8); cudaMalloc(&dout, 8);
    cudaMemset(dx, 0, n * 8);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (auto &cs : cases) {
        cudaMemcpy(dcol, cs.v.data(), nnz * 4, cudaMemcpyHostToDevice);
        for (int path = 0; path < 2; ++path) {
            for (int grid : {148 * 8, 148 * 16}) {
                float best = 1e9;
                for (int rep = 0; rep < 5; ++rep) {
                    cudaEventRecord(e0);
                    if (path == 0) gather<8, true><<<grid, 256>>>(dcol, nnz, dx, dout);
                    else gather<8, false><<<grid, 256>>>(dcol, nnz, dx, dout);
                    cudaEventRecord(e1); cudaEventSynchronize(e1);
                    float ms; cudaEventElapsedTime(&ms, e0, e1); best = std::min(best, ms);
                }
                printf("%-16s %s grid=%5d  %8.1f us  %6.2f Ggather/s\n", cs.name, path ? "ld.cg" : "ld.nc", grid,
                       best * 1e3, nnz / (best * 1e-3) / 1e9);
            }
        }
    }
    return 0;
}
