// fp64 / MUFU latency and throughput probe on the GPU box:
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 fp64_lat.cu -o fp64_lat
#include <cstdio>
#include <cuda_runtime.h>

template <int OP>
__global__ void lat(double* out, long long* cyc, double a, double b, int iters) {
    double x = a + threadIdx.x * 1e-9, y = b;
    long long t0 = clock64();
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int k = 0; k < 16; ++k) {
            if (OP == 0) x = x + y;
            else if (OP == 1) x = fma(x, y, 1e-3);
            else if (OP == 2) { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x)); x = r; }
            else if (OP == 3) x = x * y;
            else { float f = (float)x; f = f * 1.0001f + 1e-3f; x = f; }
        }
    }
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
    out[blockIdx.x * blockDim.x + threadIdx.x] = x;
}

template <int OP, int ILP>
__global__ void thr(double* out, double a, double b, int iters) {
    double x[ILP];
#pragma unroll
    for (int q = 0; q < ILP; ++q) x[q] = a + q + threadIdx.x * 1e-9;
    for (int i = 0; i < iters; ++i) {
#pragma unroll
        for (int q = 0; q < ILP; ++q) {
            if (OP == 0) x[q] = x[q] + b;
            else if (OP == 1) x[q] = fma(x[q], b, 1e-3);
            else { double r; asm volatile("rcp.approx.ftz.f64 %0, %1;" : "=d"(r) : "d"(x[q])); x[q] = r; }
        }
    }
    double s = 0;
#pragma unroll
    for (int q = 0; q < ILP; ++q) s += x[q];
    out[blockIdx.x * blockDim.x + threadIdx.x] = s;
}

int main() {
    double* out; long long* cyc;
    cudaMalloc(&out, 148 * 1024 * 8 * 8);
    cudaMalloc(&cyc, 1024 * 8);
    const char* names[] = {"DADD", "DFMA", "MUFU.RCP64H", "DMUL", "F2F+FFMA"};
    for (int op = 0; op < 5; ++op) {
        long long h[1];
        int iters = 1000;
        for (int rep = 0; rep < 2; ++rep) {
            switch (op) {
                case 0: lat<0><<<1, 32>>>(out, cyc, 1.0, 1e-9, iters); break;
                case 1: lat<1><<<1, 32>>>(out, cyc, 1.0, 0.999, iters); break;
                case 2: lat<2><<<1, 32>>>(out, cyc, 1.5, 0.0, iters); break;
                case 3: lat<3><<<1, 32>>>(out, cyc, 1.0, 0.999999, iters); break;
                default: lat<4><<<1, 32>>>(out, cyc, 1.0, 0.0, iters); break;
            }
            cudaDeviceSynchronize();
        }
        cudaMemcpy(h, cyc, 8, cudaMemcpyDeviceToHost);
        printf("latency %-12s %.1f cycles\n", names[op], (double)h[0] / (iters * 16));
    }
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0); cudaEventCreate(&e1);
    int sms = 148;
    for (int op = 0; op < 3; ++op) {
        for (int warps : {4, 8, 16, 32}) {
            const int iters = 4000;
            float ms = 0;
            for (int rep = 0; rep < 2; ++rep) {
                cudaEventRecord(e0);
                if (op == 0) thr<0, 8><<<sms, warps * 32>>>(out, 1.0, 1e-9, iters);
                else if (op == 1) thr<1, 8><<<sms, warps * 32>>>(out, 1.0, 0.999, iters);
                else thr<2, 8><<<sms, warps * 32>>>(out, 1.5, 0.0, iters);
                cudaEventRecord(e1);
                cudaEventSynchronize(e1);
                cudaEventElapsedTime(&ms, e0, e1);
            }
            double ops = (double)sms * warps * 32 * iters * 8;
            printf("throughput %-12s warps/SM=%2d  %.2f Gop/s  = %.1f lane-ops/clk/SM (@1.965GHz)\n",
                   names[op], warps, ops / ms / 1e6, ops / (ms * 1e-3) / sms / 1.965e9);
        }
    }
    return 0;
}
