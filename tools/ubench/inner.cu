// Inner-loop microbenchmark of the BiQGEMM fast path (one SM, keys+LUT in smem).
#include <cstdio>
#include <cstdint>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t off7(uint32_t w, int bi, uint32_t lo) {
    const int s = 8 * bi - 7;
    const uint32_t v = s >= 0 ? (w >> s) : (w << (-s));
    return (v & 0x7f80u) | lo;
}

template <int MODE>
__global__ void __launch_bounds__(1024) inner(float* out, long long* cyc, int iters) {
    __shared__ __align__(16) float lut[256 * 32];
    __shared__ __align__(16) uint32_t keys[16][256];  // 16 chunks x 1 KB
    for (int i = threadIdx.x; i < 256 * 32; i += blockDim.x) lut[i] = (float)(i % 97);
    for (int i = threadIdx.x; i < 16 * 256; i += blockDim.x) ((uint32_t*)keys)[i] = i * 2654435761u;
    __syncthreads();
    const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
    const uint32_t lo = lane * 4;
    const char* lutc = (const char*)lut;
    float acc = 0.f;
    long long t0 = clock64();
    for (int it = 0; it < iters; ++it) {
        const uint32_t* kc = keys[(it + warp) & 15];
        uint4 a = *(const uint4*)(kc + lane * 4);
        uint4 b = *(const uint4*)(kc + 128 + lane * 4);
        uint32_t w[8] = {a.x, a.y, a.z, a.w, b.x, b.y, b.z, b.w};
        float v[32];
#pragma unroll
        for (int wi = 0; wi < 8; ++wi)
#pragma unroll
            for (int bi = 0; bi < 4; ++bi) {
                if (MODE == 2) v[wi * 4 + bi] = __uint_as_float(off7(w[wi], bi, lo));
                else v[wi * 4 + bi] = *(const float*)(lutc + off7(w[wi], bi, lo));
            }
        if (MODE == 1) {  // no butterfly: plain sum
#pragma unroll
            for (int s = 1; s < 32; ++s) v[0] += v[s];
        } else {
#pragma unroll
            for (int hw = 16; hw >= 1; hw >>= 1)
#pragma unroll
                for (int s = 0; s < hw; ++s) v[s] += __shfl_xor_sync(0xffffffffu, v[s + hw], hw);
        }
        acc += v[0];
    }
    long long t1 = clock64();
    out[blockIdx.x * blockDim.x + threadIdx.x] = acc;
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main() {
    float* out; long long* cyc;
    cudaMalloc(&out, 4 << 20); cudaMallocManaged(&cyc, 8 * 1024);
    const int iters = 2000;
    const char* names[3] = {"gather+butterfly", "gather+serial-sum", "no-gather+butterfly"};
    for (int mode = 0; mode < 3; ++mode) {
        for (int warps : {2, 4, 8, 16, 32}) {
            auto k = mode == 0 ? inner<0> : (mode == 1 ? inner<1> : inner<2>);
            k<<<1, warps * 32>>>(out, cyc, iters);
            k<<<1, warps * 32>>>(out, cyc, iters);
            cudaDeviceSynchronize();
            double per_chunk_sm = (double)cyc[0] / iters / warps;
            printf("%-22s warps %2d: %.1f cycles per chunk per warp, %.1f cycles per chunk per SM (LDS bound 32)\n",
                   names[mode], warps, (double)cyc[0] / iters, per_chunk_sm);
        }
    }
    return 0;
}
