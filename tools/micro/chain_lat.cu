// Dependent-latency micro-benchmark (dev tool, GPU box): one warp alone on an SM, clock64
// around N unrolled iterations of
//   fadd   : x = x + c                        (FADD -> FADD)
//   fmul   : x = x * c                        (FMUL -> FMUL)
//   step   : the dwell step of csrc/dwell.cuh (3 FMUL + 2 FADD + 1 FFMA-imm)
//   step2  : two independent dwell orbits interleaved in one thread
//   stepx2 : the packed step (FMUL2/FADD2/FFMA2 on float2 halves), one packed orbit pair
// Prints cycles per iteration.  Build: nvcc -gencode arch=compute_100a,code=sm_100a -O3
//   -fmad=false -o /tmp/chain_lat tools/micro/chain_lat.cu
#include <cstdio>
#include <cstdint>

#define N 4096

__device__ __forceinline__ void step(float &x, float &y, float &x2, float &y2, float cr, float ci)
{
    float xy = __fmul_rn(x, y);
    x = __fadd_rn(__fsub_rn(x2, y2), cr);
    y = __fmaf_rn(xy, 2.0f, ci);
    x2 = __fmul_rn(x, x);
    y2 = __fmul_rn(y, y);
}

__global__ void k(int mode, float cr, float ci, float *out, long long *cyc)
{
    float x = 0.f, y = 0.f, x2 = 0.f, y2 = 0.f;
    float u = 0.f, v = 0.f, u2 = 0.f, v2 = 0.f;
    float a = cr + threadIdx.x * 1e-9f;
    __syncwarp();
    long long t0 = clock64();
    if (mode == 0) {
#pragma unroll 64
        for (int i = 0; i < N; ++i)
            a = __fadd_rn(a, ci);
        x = a;
    } else if (mode == 1) {
#pragma unroll 64
        for (int i = 0; i < N; ++i)
            a = __fmul_rn(a, ci);
        x = a;
    } else if (mode == 2) {
#pragma unroll 32
        for (int i = 0; i < N; ++i)
            step(x, y, x2, y2, a, ci);
    } else if (mode == 3) {
        float b = a + 1e-7f;
#pragma unroll 32
        for (int i = 0; i < N; ++i) {
            step(x, y, x2, y2, a, ci);
            step(u, v, u2, v2, b, ci);
        }
        x += u;
    }
    long long t1 = clock64();
    out[threadIdx.x] = x + y + x2 + y2;
    if (threadIdx.x == 0)
        *cyc = t1 - t0;
}

int main()
{
    float *out;
    long long *cyc, h;
    cudaMalloc(&out, 4096 * 4);
    cudaMalloc(&cyc, 8);
    const char *names[] = {"fadd_chain", "fmul_chain", "dwell_step", "dwell_step_x2_orbits"};
    for (int m = 0; m < 4; ++m) {
        for (int rep = 0; rep < 3; ++rep) {
            k<<<1, 32>>>(m, -0.1f, 0.1f, out, cyc);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("{\"mode\": \"%s\", \"warps_per_block\": 1, \"cycles_per_iter\": %.2f}\n", names[m], (double)h / N);
    }
    // one block of w warps on one SM (w / 4 warps per sub-partition): the dwell step
    for (int w = 2; w <= 32; w *= 2) {
        for (int rep = 0; rep < 3; ++rep) {
            k<<<1, 32 * w>>>(2, -0.1f, 0.1f, out, cyc);
            cudaMemcpy(&h, cyc, 8, cudaMemcpyDeviceToHost);
        }
        printf("{\"mode\": \"dwell_step\", \"warps_per_block\": %d, \"cycles_per_iter\": %.2f}\n", w, (double)h / N);
    }
    return 0;
}
