// Does a key stream fetched through the TEXTURE pipe (tex1Dfetch) or plain
// LDG compete with a conflict-free shared-memory LUT gather for the SM's
// L1TEX data pipe?  One CTA per SM, NG gather warps (PRMT + LDS + FADD on
// register-generated keys, the stream kernel's inner loop) and NS stream
// warps (HBM -> registers, 2 GiB buffer, XOR sink).  Modes: gather only,
// stream only, both.  If "both" takes max(alone) the pipes are independent.
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }

template <int SMODE>  // 0 tex, 1 ldg.nc.L1::no_allocate v4, 2 ldg v8 (256-bit)
__device__ __forceinline__ void stream_part(cudaTextureObject_t tex, const uint4* buf, long long per_warp_u4,
                                            long long base_u4, int lane, uint32_t& sink) {
    const long long n = per_warp_u4;
    for (long long i = 0; i < n; i += 32 * 8) {
        uint4 v[8];
#pragma unroll
        for (int u = 0; u < 8; ++u) {
            const long long idx = base_u4 + i + u * 32 + lane;
            if constexpr (SMODE == 0) {
                v[u] = tex1Dfetch<uint4>(tex, (int)idx);
            } else {
                asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
                             : "=r"(v[u].x), "=r"(v[u].y), "=r"(v[u].z), "=r"(v[u].w)
                             : "l"(buf + idx));
            }
        }
#pragma unroll
        for (int u = 0; u < 8; ++u) sink ^= v[u].x ^ v[u].y ^ v[u].z ^ v[u].w;
    }
}

template <int SMODE>
__global__ void __launch_bounds__(1024, 1) k(cudaTextureObject_t tex, const uint4* buf, long long per_cta_u4,
                                             int ng, int ns, int gather_iters, float* out, long long* cyc) {
    extern __shared__ __align__(1024) unsigned char sm[];
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    float* lut = reinterpret_cast<float*>(sm);
    for (int i = threadIdx.x; i < 64 * 256; i += blockDim.x) lut[i] = (float)(i % 97);
    __syncthreads();
    long long t0 = clock64();
    if (warp < ng) {
        uint32_t rot[8];
#pragma unroll
        for (int q = 0; q < 8; ++q) {
            rot[q] = 0;
#pragma unroll
            for (int b = 0; b < 4; ++b) rot[q] |= ((uint32_t)((lane + 4 * q + b) & 31) * 4u) << (8 * b);
        }
        uint32_t s = 0x9E3779B9u * (threadIdx.x + 1) + blockIdx.x;
        float acc0 = 0.f, acc1 = 0.f, acc2 = 0.f, acc3 = 0.f;
        const uint32_t base = smem_u32(lut);
        for (int it = 0; it < gather_iters; ++it) {
            uint32_t w[8];
#pragma unroll
            for (int q = 0; q < 8; ++q) { s = s * 1664525u + 1013904223u; w[q] = s; }
#pragma unroll
            for (int q = 0; q < 8; ++q) {
#pragma unroll
                for (int bi = 0; bi < 4; ++bi) {
                    uint32_t off;
                    asm("prmt.b32 %0, %1, %2, %3;" : "=r"(off) : "r"(rot[q]), "r"(w[q]), "r"(0x8840u + 0x11u * bi));
                    float e;
                    asm volatile("ld.shared.f32 %0, [%1];" : "=f"(e) : "r"(base + off));
                    if (bi == 0) acc0 += e; else if (bi == 1) acc1 += e; else if (bi == 2) acc2 += e; else acc3 += e;
                }
            }
        }
        out[blockIdx.x * 1024 + threadIdx.x] = acc0 + acc1 + acc2 + acc3;
    } else if (warp < ng + ns) {
        uint32_t sink = 0;
        const long long per_warp = per_cta_u4 / ns;
        stream_part<SMODE>(tex, buf, per_warp, blockIdx.x * per_cta_u4 + (warp - ng) * per_warp, lane, sink);
        out[blockIdx.x * 1024 + threadIdx.x] = (float)sink;
    }
    __syncthreads();
    long long t1 = clock64();
    if (threadIdx.x == 0) cyc[blockIdx.x] = t1 - t0;
}

int main(int argc, char** argv) {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = 2ull << 30;
    uint4* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    float* out;
    long long* cyc;
    cudaMalloc(&out, (size_t)sms * 1024 * 4);
    cudaMallocManaged(&cyc, sms * 8);
    // texture on a linear buffer: max 2^27 texels -> 2 GiB of uint4
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = buf;
    rd.res.linear.desc = cudaCreateChannelDesc(32, 32, 32, 32, cudaChannelFormatKindUnsigned);
    rd.res.linear.sizeInBytes = bytes;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t tex = 0;
    if (cudaCreateTextureObject(&tex, &rd, &td, nullptr) != cudaSuccess) { printf("tex create failed\n"); return 1; }
    const int smem = (argc > 1 ? atoi(argv[1]) : 64) * 1024;
    cudaFuncSetAttribute(k<0>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaFuncSetAttribute(k<1>, cudaFuncAttributeMaxDynamicSharedMemorySize, smem);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const long long per_cta_u4 = (long long)(bytes / 16 / sms) / 8192 * 8192;
    const char* sn[2] = {"tex1Dfetch", "ldg.nc.v4"};
    for (int smode = 0; smode < (argc > 2 ? atoi(argv[2]) : 2); ++smode) {
        for (int ns : {4, 8}) {
            for (int ng : {16, 24}) {
                for (int mode = 0; mode < 3; ++mode) {
                    // gather iterations sized so gather alone ~ stream alone at ~6 TB/s
                    const int gi = 2400;
                    const int g = mode == 1 ? 0 : ng, s = mode == 0 ? 0 : ns;
                    auto kern = smode == 0 ? k<0> : k<1>;
                    kern<<<sms, (ng + ns) * 32, smem>>>(tex, buf, per_cta_u4, g, s, gi, out, cyc);
                    cudaEventRecord(e0);
                    kern<<<sms, (ng + ns) * 32, smem>>>(tex, buf, per_cta_u4, g, s, gi, out, cyc);
                    cudaEventRecord(e1);
                    cudaError_t err = cudaEventSynchronize(e1);
                    if (err != cudaSuccess) { printf("err %s\n", cudaGetErrorString(err)); return 1; }
                    float ms = 0;
                    cudaEventElapsedTime(&ms, e0, e1);
                    const double lds_wf = (double)g * gi * 32 * sms;  // wavefronts (conflict-free LDS.32)
                    const double sbytes = s ? (double)per_cta_u4 * 16 * sms : 0;
                    double cmax = 0;
                    for (int i = 0; i < sms; ++i) cmax = cyc[i] > cmax ? cyc[i] : cmax;
                    printf("%-10s ns=%d ng=%2d mode=%s: %.3f ms  LDS wf/clk/SM %.3f  stream %.0f GB/s (%.1f B/clk/SM)\n", sn[smode],
                           ns, ng, mode == 0 ? "gather" : (mode == 1 ? "stream" : "both  "), ms,
                           lds_wf / sms / cmax, sbytes / ms / 1e6, sbytes / sms / cmax);
                }
            }
        }
    }
    return 0;
}
