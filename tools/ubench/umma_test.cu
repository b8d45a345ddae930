// Unit test of the tcgen05 kind::tf32 helpers (afam_umma.cuh): D(M x N) =
// A(M x K) B(N x K)^T in 3xTF32, K-major no-swizzle operands, read back
// through TMEM; compared with a float64 host product.
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <vector>

#include "../../paper_2409_00184_b200/csrc/afam_umma.cuh"
using namespace afam;

template <int M, int N, int K>
__global__ void umma_kernel(const float *A, const float *B, float *D, int mode) {
    extern __shared__ __align__(128) unsigned char smem[];
    float *ah = (float *)smem, *al = ah + M * K, *bh = al + M * K, *bl = bh + N * K;
    __shared__ uint64_t bar;
    __shared__ uint32_t tbase;
    // canonical K-major panels: ((k/4)*R + r)*4 + k%4 (floats)
    for (int i = threadIdx.x; i < M * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        float h, l;
        umma::split_tf32(A[i], h, l);
        ah[((k / 4) * M + r) * 4 + k % 4] = h;
        al[((k / 4) * M + r) * 4 + k % 4] = l;
    }
    for (int i = threadIdx.x; i < N * K; i += blockDim.x) {
        const int r = i / K, k = i % K;
        float h, l;
        umma::split_tf32(B[i], h, l);
        bh[((k / 4) * N + r) * 4 + k % 4] = h;
        bl[((k / 4) * N + r) * 4 + k % 4] = l;
    }
    if (threadIdx.x == 0) {
        asm volatile("mbarrier.init.shared::cta.b64 [%0], 1;" ::"r"(umma::smem_addr(&bar)));
        asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    }
    if (threadIdx.x < 32) umma::tmem_alloc(&tbase, 64 < N ? 128 : 64);
    umma::fence_async_smem();
    umma::fence_before_sync();
    __syncthreads();
    umma::fence_after_sync();
    const uint32_t t0 = tbase;
    if (threadIdx.x == 0) {
        constexpr uint32_t idesc = umma::idesc_tf32(M, N);
        for (int ks = 0; ks < K / 8; ks++) {
            const uint32_t off_a = ks * 2 * M * 16, off_b = ks * 2 * N * 16;
            const uint64_t dah = umma::desc_kmajor(umma::smem_addr(ah) + off_a, M * 16, 128);
            const uint64_t dal = umma::desc_kmajor(umma::smem_addr(al) + off_a, M * 16, 128);
            const uint64_t dbh = umma::desc_kmajor(umma::smem_addr(bh) + off_b, N * 16, 128);
            const uint64_t dbl = umma::desc_kmajor(umma::smem_addr(bl) + off_b, N * 16, 128);
            umma::mma_tf32(t0, dah, dbh, idesc, ks > 0);
            if (mode == 3) {
                umma::mma_tf32(t0, dal, dbh, idesc, true);
                umma::mma_tf32(t0, dah, dbl, idesc, true);
            }
        }
        umma::commit(&bar);
    }
    // wait for the MMAs
    asm volatile(
        "{\n\t.reg .pred p;\nW_%=:\n\tmbarrier.try_wait.parity.shared::cta.b64 p, [%0], 0;\n\t@!p bra W_%=;\n}" ::"r"(
            umma::smem_addr(&bar))
        : "memory");
    umma::fence_after_sync();
    const int w = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (w < 4) {
        for (int c = 0; c < N; c += 16) {
            float v[16];
            umma::tmem_ld16(t0 + ((uint32_t)(32 * w) << 16) + c, v);
            int row;
            if (M == 128) row = 32 * w + lane;
            else row = lane < 16 ? 16 * w + lane : -1;
            if (row >= 0)
                for (int q = 0; q < 16; q++) D[row * N + c + q] = v[q];
        }
    }
    umma::fence_before_sync();
    __syncthreads();
    if (threadIdx.x < 32) umma::tmem_dealloc(t0, 64 < N ? 128 : 64);
}

template <int M, int N, int K>
int run(int mode) {
    std::vector<float> A(M * K), B(N * K), D(M * N, 0.f);
    srand(1);
    for (auto &x : A) x = (float)rand() / RAND_MAX * 2 - 1;
    for (auto &x : B) x = (float)rand() / RAND_MAX;
    float *dA, *dB, *dD;
    cudaMalloc(&dA, A.size() * 4); cudaMalloc(&dB, B.size() * 4); cudaMalloc(&dD, D.size() * 4);
    cudaMemcpy(dA, A.data(), A.size() * 4, cudaMemcpyHostToDevice);
    cudaMemcpy(dB, B.data(), B.size() * 4, cudaMemcpyHostToDevice);
    cudaMemset(dD, 0xff, D.size() * 4);
    const size_t sm = (size_t)(2 * M * K + 2 * N * K) * 4;
    cudaFuncSetAttribute(umma_kernel<M, N, K>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm);
    umma_kernel<M, N, K><<<1, 128, sm>>>(dA, dB, dD, mode);
    cudaError_t e = cudaDeviceSynchronize();
    if (e != cudaSuccess) { printf("M=%d N=%d K=%d: CUDA error %s\n", M, N, K, cudaGetErrorString(e)); return 1; }
    cudaMemcpy(D.data(), dD, D.size() * 4, cudaMemcpyDeviceToHost);
    double maxerr = 0, maxref = 0;
    for (int i = 0; i < M; i++)
        for (int j = 0; j < N; j++) {
            double s = 0;
            for (int k = 0; k < K; k++) s += (double)A[i * K + k] * B[j * K + k];
            maxerr = fmax(maxerr, fabs(s - D[i * N + j]));
            maxref = fmax(maxref, fabs(s));
            if (!(fabs(s - D[i * N + j]) < 1e-2) && i < 2) printf("  D[%d][%d] = %g want %g\n", i, j, D[i * N + j], s);
        }
    printf("M=%d N=%d K=%d %s: max |err| %.3e (max |D| %.3f)\n", M, N, K, mode == 3 ? "3xTF32" : "1xTF32", maxerr,
           maxref);
    return 0;
}

int main() {
    run<128, 64, 16>(1);
    run<128, 64, 16>(3);
    run<64, 64, 72>(1);
    run<64, 64, 72>(3);
    run<64, 16, 24>(3);
    run<128, 16, 72>(3);
    return 0;
}
