// Texture-fetch streaming rate vs access pattern (what the grouped tex form
// does vs what tools/ubench/lsu_tex.cu does).  One CTA per SM, NW warps,
// each fetches "units" of B KiB (2*B TLD.128 per lane) with UD units in
// registers, XOR sink.  Knobs:
//   pattern 0: warp w streams its own contiguous slice of the CTA's range
//   pattern 1: units of the CTA's range dealt round-robin to the warps (the kernel)
//   ntex: the buffer is split into ntex texture objects ("calls"); a unit
//         uses the object that covers it (handle from a kernel-param array)
#include <cstdint>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

struct Args {
    unsigned long long tex[512];
    long long units_per_tex;  // units covered by one texture
    long long total_units;
    int nw, pattern, uniform;
};

template <int B, int UD>
__global__ void __launch_bounds__(1024, 1) k(const __grid_constant__ Args A, unsigned* out) {
    const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
    if (warp >= A.nw) return;
    const long long U0 = blockIdx.x * A.total_units / gridDim.x, U1 = (blockIdx.x + 1) * A.total_units / gridDim.x;
    const long long n = U1 - U0;
    long long first, step, cnt;
    if (A.pattern == 0) {
        const long long per = n / A.nw;
        first = U0 + warp * per;
        step = 1;
        cnt = per;
    } else {
        first = U0 + warp;
        step = A.nw;
        cnt = n > warp ? (n - warp + A.nw - 1) / A.nw : 0;
    }
    uint4 K[UD][B][2];
    unsigned h = 0;
    auto fetch = [&](long long u, uint4 (&kk)[B][2]) {
        const long long ti = u / A.units_per_tex;
        const cudaTextureObject_t t = A.uniform ? A.tex[0] : A.tex[ti];
        const int base = static_cast<int>((u - ti * A.units_per_tex) * B * 64) + lane;
#pragma unroll
        for (int i = 0; i < B; ++i) {
            kk[i][0] = tex1Dfetch<uint4>(t, base + i * 64);
            kk[i][1] = tex1Dfetch<uint4>(t, base + i * 64 + 32);
        }
    };
#pragma unroll
    for (int d = 0; d < UD; ++d)
        if (d < cnt) fetch(first + d * step, K[d]);
    for (long long k0 = 0; k0 < cnt; k0 += UD) {
#pragma unroll
        for (int d = 0; d < UD; ++d) {
            if (k0 + d < cnt) {
#pragma unroll
                for (int i = 0; i < B; ++i) h ^= K[d][i][0].x ^ K[d][i][0].w ^ K[d][i][1].y ^ K[d][i][1].z;
                if (k0 + d + UD < cnt) fetch(first + (k0 + d + UD) * step, K[d]);
            }
        }
    }
    out[blockIdx.x * 1024 + threadIdx.x] = h;
}

int main() {
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    const size_t bytes = 1ull << 30;
    char* buf;
    cudaMalloc(&buf, bytes);
    cudaMemset(buf, 1, bytes);
    unsigned* out;
    cudaMalloc(&out, (size_t)sms * 1024 * 4);
    cudaEvent_t e0, e1;
    cudaEventCreate(&e0);
    cudaEventCreate(&e1);
    const int B = 3;
    const long long unit = B * 1024;
    for (int ntex : {1, 128}) for (int uni : {0, 1}) {
        if (uni && ntex > 1) continue;
        Args A = {};
        const long long per_tex_bytes = (bytes / ntex) / unit * unit;
        for (int i = 0; i < ntex; ++i) {
            cudaResourceDesc rd = {};
            rd.resType = cudaResourceTypeLinear;
            rd.res.linear.devPtr = buf + i * per_tex_bytes;
            rd.res.linear.desc = cudaCreateChannelDesc(32, 32, 32, 32, cudaChannelFormatKindUnsigned);
            rd.res.linear.sizeInBytes = per_tex_bytes;
            cudaTextureDesc td = {};
            td.readMode = cudaReadModeElementType;
            cudaTextureObject_t t;
            cudaCreateTextureObject(&t, &rd, &td, nullptr);
            A.tex[i] = t;
        }
        A.units_per_tex = per_tex_bytes / unit;
        A.total_units = A.units_per_tex * ntex;
        for (int pattern : {0, 1})
            for (int nw : {8, 16, 24}) {
                for (int ud : {1, 2, 3}) {
                    A.nw = nw;
                    A.pattern = pattern;
                    A.uniform = uni;
                    auto kern = ud == 1 ? k<B, 1> : (ud == 2 ? k<B, 2> : k<B, 3>);
                    kern<<<sms, nw * 32>>>(A, out);
                    cudaEventRecord(e0);
                    kern<<<sms, nw * 32>>>(A, out);
                    cudaEventRecord(e1);
                    if (cudaEventSynchronize(e1) != cudaSuccess) { printf("error\n"); return 1; }
                    float ms;
                    cudaEventElapsedTime(&ms, e0, e1);
                    printf("uniform %d ntex %3d pattern %d nw %2d ud %d: %7.0f GB/s\n", uni, ntex, pattern, nw, ud,
                           A.total_units * unit / ms / 1e6);
                }
            }
    }
    return 0;
}
