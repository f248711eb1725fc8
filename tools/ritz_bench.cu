// Diagnostic microbenchmark (not part of the product): ritz_warp alone on one warp.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -std=c++17 -I. tools/ritz_bench.cu -o /tmp/ritz_bench
#include "../paper_1501_06211_b200/csrc/kernels_prec_coop.cu"
#include <cstdio>

using namespace de;

__global__ void k_ritz(const double* A, const double* B, const double* wr, int n, double* coef,
                       unsigned long long* tm, long long* cyc) {
    extern __shared__ double ws[];
    double* R = ws;
    double* Cm = R + KMAX * (KMAX + 1);
    double* V = Cm + KMAX * (KMAX + 1);
    double* X = V + KMAX * (KMAX + 1);
    double* rot = X + KMAX * (KMAX + 1);
    int* rpq = reinterpret_cast<int*>(rot + KMAX);
    const long long t0 = clock64();
    ritz_warp(A, B, wr, n, false, 0.5, coef, R, Cm, V, X, rot, rpq, tm);
    if (threadIdx.x == 0) *cyc = clock64() - t0;
}

int main() {
    const int n = 10;
    double hA[KMAX * KMAX] = {}, hB[KMAX * KMAX] = {}, hw[KMAX] = {};
    unsigned s = 12345;
    auto rnd = [&]() { s = s * 1664525u + 1013904223u; return (s >> 8) / double(1 << 24) - 0.5; };
    double G[KMAX][KMAX];
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) G[i][j] = rnd();
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < n; ++j) {
            double t = 0;
            for (int k = 0; k < n; ++k) t += G[i][k] * G[j][k];
            hA[i * KMAX + j] = t + (i == j ? 1e-3 * pow(10.0, i % 6) : 0.0);
            hB[i * KMAX + j] = (i == j ? 1.0 : 1e-9 * rnd());
        }
    for (int i = 0; i < n; ++i) hB[i * KMAX + i] += 0.0;
    for (int i = 0; i < n; ++i)
        for (int j = 0; j < i; ++j) hB[i * KMAX + j] = hB[j * KMAX + i];
    for (int i = 0; i < n; ++i) hw[i] = rnd();
    double *A, *B, *w, *coef;
    unsigned long long* tm;
    long long* cyc;
    cudaMalloc(&A, sizeof hA); cudaMalloc(&B, sizeof hB); cudaMalloc(&w, sizeof hw);
    cudaMalloc(&coef, KMAX * 8); cudaMalloc(&tm, 16 * 8); cudaMalloc(&cyc, 8);
    cudaMemcpy(A, hA, sizeof hA, cudaMemcpyHostToDevice);
    cudaMemcpy(B, hB, sizeof hB, cudaMemcpyHostToDevice);
    cudaMemcpy(w, hw, sizeof hw, cudaMemcpyHostToDevice);
    const size_t smem = (4 * KMAX * (KMAX + 1) + 2 * KMAX + 4 * KMAX) * 8;
    for (int rep = 0; rep < 3; ++rep) {
        k_ritz<<<1, 32, smem>>>(A, B, w, n, coef, tm, cyc);
        cudaDeviceSynchronize();
        unsigned long long t[16];
        long long c;
        cudaMemcpy(t, tm, sizeof t, cudaMemcpyDeviceToHost);
        cudaMemcpy(&c, cyc, 8, cudaMemcpyDeviceToHost);
        double cf[KMAX];
        cudaMemcpy(cf, coef, sizeof cf, cudaMemcpyDeviceToHost);
        printf("coef0..2 %.15e %.15e %.15e\n", cf[0], cf[1], cf[2]);
        printf("err %s cycles %lld setup %.1f us jacobi %.1f us sweeps %llu final %.1f us\n",
               cudaGetErrorString(cudaGetLastError()), c, (t[1] - t[0]) / 1e3, (t[2] - t[1]) / 1e3, t[4],
               (t[3] - t[2]) / 1e3);
    }
    return 0;
}
