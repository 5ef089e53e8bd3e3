// Can ONE linear texture object span several separate allocations (so a
// grouped launch needs a single, warp-uniform texture handle)?
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

__global__ void fetch(cudaTextureObject_t t, const long long* offs, int n, unsigned* out) {
    const int i = blockIdx.x;
    if (i < n) {
        uint4 v = tex1Dfetch<uint4>(t, static_cast<int>(offs[i]) + threadIdx.x);
        out[i * 32 + threadIdx.x] = v.x;
    }
}

int main() {
    int w = 0, al = 0, w2 = 0;
    cudaDeviceGetAttribute(&w, cudaDevAttrMaxTexture1DLinearWidth, 0);
    cudaDeviceGetAttribute(&al, cudaDevAttrTextureAlignment, 0);
    cudaDeviceGetAttribute(&w2, cudaDevAttrMaxTexture2DLinearWidth, 0);
    printf("max 1D linear width %d texels, texture alignment %d, 2D linear width %d\n", w, al, w2);
    const int n = 6;
    char* b[n];
    void* gap = nullptr;
    for (int i = 0; i < n; ++i) {
        cudaMalloc(&b[i], 8 << 20);
        cudaMemset(b[i], i + 1, 8 << 20);
        if (i == 2) { cudaMalloc(&gap, 1ull << 30); }
    }
    cudaFree(gap);  // leaves an unmapped hole between b[2] and b[3] (maybe)
    uintptr_t lo = ~0ull, hi = 0;
    for (int i = 0; i < n; ++i) {
        printf("buf %d at %p\n", i, b[i]);
        lo = (uintptr_t)b[i] < lo ? (uintptr_t)b[i] : lo;
        hi = (uintptr_t)b[i] + (8 << 20) > hi ? (uintptr_t)b[i] + (8 << 20) : hi;
    }
    lo &= ~(uintptr_t)(al - 1);
    printf("span %.1f MB\n", (hi - lo) / 1e6);
    cudaResourceDesc rd = {};
    rd.resType = cudaResourceTypeLinear;
    rd.res.linear.devPtr = (void*)lo;
    rd.res.linear.desc = cudaCreateChannelDesc(32, 32, 32, 32, cudaChannelFormatKindUnsigned);
    rd.res.linear.sizeInBytes = hi - lo;
    cudaTextureDesc td = {};
    td.readMode = cudaReadModeElementType;
    cudaTextureObject_t t = 0;
    cudaError_t e = cudaCreateTextureObject(&t, &rd, &td, nullptr);
    printf("create spanning texture: %s\n", cudaGetErrorString(e));
    if (e != cudaSuccess) return 0;
    long long* offs;
    unsigned* out;
    cudaMallocManaged(&offs, n * 8);
    cudaMallocManaged(&out, n * 32 * 4);
    for (int i = 0; i < n; ++i) offs[i] = ((uintptr_t)b[i] - lo) / 16 + 1000;
    fetch<<<n, 32>>>(t, offs, n, out);
    e = cudaDeviceSynchronize();
    printf("fetch: %s\n", cudaGetErrorString(e));
    for (int i = 0; i < n; ++i) printf("buf %d value %08x (expect %02x%02x%02x%02x)\n", i, out[i * 32], i + 1, i + 1, i + 1, i + 1);
    // a range > max width
    rd.res.linear.sizeInBytes = (size_t)w * 16 + 16;
    e = cudaCreateTextureObject(&t, &rd, &td, nullptr);
    printf("create over-wide texture: %s\n", cudaGetErrorString(e));
    return 0;
}
