// Micro-benchmarks for the fp64 score path on B200 (sm_100a):
// DFMA latency (dependent chain), DFMA throughput, DADD latency,
// F2F.F64.F32 throughput, double sqrt/div latency.
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o ubench_fp64 tools/ubench_fp64.cu
#include <cstdio>
#include <cuda_runtime.h>

__global__ void dfma_lat(double* out, long long* cyc, int n) {
    double a = out[0], b = out[1], c = out[2];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        c = fma(a, b, c);
        c = fma(a, b, c);
        c = fma(a, b, c);
        c = fma(a, b, c);
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[3] = c; }
}

__global__ void dadd_lat(double* out, long long* cyc, int n) {
    double a = out[0], c = out[2];
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        c = c + a; c = c + a; c = c + a; c = c + a;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[3] = c; }
}

__global__ void sqrtdiv_lat(double* out, long long* cyc, int n) {
    double c = out[0] + 2.0;
    long long t0 = clock64();
    for (int i = 0; i < n; ++i) {
        c = sqrt(c) + 1.5;
        c = 7.0 / c + 2.0;
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) { cyc[0] = t1 - t0; out[3] = c; }
}

template <int K>
__global__ void dfma_tput(double* out, int n) {
    double a = out[0], b = out[1];
    double c[K];
#pragma unroll
    for (int k = 0; k < K; ++k) c[k] = out[2] + k;
    for (int i = 0; i < n; ++i) {
#pragma unroll
        for (int k = 0; k < K; ++k) c[k] = fma(a, b, c[k]);
    }
    double s = 0;
#pragma unroll
    for (int k = 0; k < K; ++k) s += c[k];
    if (s == 12345.0) out[4] = s;
}

__global__ void f2f_tput(double* out, float* in, int n) {
    float x0 = in[threadIdx.x & 31], x1 = x0 + 1, x2 = x0 + 2, x3 = x0 + 3;
    double s0 = 0, s1 = 0, s2 = 0, s3 = 0;
    for (int i = 0; i < n; ++i) {
        s0 += (double)x0; s1 += (double)x1; s2 += (double)x2; s3 += (double)x3;
        x0 += 1.0f; x1 += 1.0f; x2 += 1.0f; x3 += 1.0f;
    }
    if (s0 + s1 + s2 + s3 == 1.0) out[5] = s0;
}

int main() {
    double* d; long long* c; float* f;
    cudaMalloc(&d, 64); cudaMalloc(&c, 64); cudaMalloc(&f, 4096);
    double h[8] = {1.0000001, 0.9999999, 0.5, 0, 0, 0, 0, 0};
    cudaMemcpy(d, h, 64, cudaMemcpyHostToDevice);
    cudaMemset(f, 0, 4096);
    int n = 4096;
    long long cy;
    dfma_lat<<<1, 32>>>(d, c, n); cudaDeviceSynchronize();
    dfma_lat<<<1, 32>>>(d, c, n); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("DFMA latency: %.2f cycles\n", (double)cy / (4.0 * n));
    dadd_lat<<<1, 32>>>(d, c, n); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("DADD latency: %.2f cycles\n", (double)cy / (4.0 * n));
    sqrtdiv_lat<<<1, 32>>>(d, c, 1024); cudaMemcpy(&cy, c, 8, cudaMemcpyDeviceToHost);
    printf("sqrt+add+div+add latency: %.2f cycles\n", (double)cy / 1024.0);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int clk; cudaDeviceGetAttribute(&clk, cudaDevAttrClockRate, 0);
    cudaEvent_t e0, e1; cudaEventCreate(&e0); cudaEventCreate(&e1);
    for (int warps : {4, 8, 16, 32}) {
        dfma_tput<8><<<sms * 4, warps * 8>>>(d, 1000);
        cudaEventRecord(e0);
        dfma_tput<8><<<sms * 4, warps * 8>>>(d, 20000);
        cudaEventRecord(e1); cudaEventSynchronize(e1);
        float ms; cudaEventElapsedTime(&ms, e0, e1);
        double ops = (double)sms * 4 * warps * 8 * 20000.0 * 8;
        printf("DFMA tput (%d thr/blk, 4 blk/SM): %.2f T/s = %.1f per clk per SM @%d MHz\n", warps * 8, ops / ms / 1e9,
               ops / (ms * 1e-3) / sms / (clk * 1e3), clk / 1000);
    }
    f2f_tput<<<sms * 8, 256>>>(d, f, 1000);
    cudaEventRecord(e0);
    f2f_tput<<<sms * 8, 256>>>(d, f, 20000);
    cudaEventRecord(e1); cudaEventSynchronize(e1);
    float ms; cudaEventElapsedTime(&ms, e0, e1);
    double ops = (double)sms * 8 * 256 * 20000.0 * 4;
    printf("F2F.F64.F32 (+DADD) tput: %.2f T/s = %.1f per clk per SM\n", ops / ms / 1e9, ops / (ms * 1e-3) / sms / (clk * 1e3));
    printf("%s\n", cudaGetErrorString(cudaGetLastError()));
    return 0;
}
