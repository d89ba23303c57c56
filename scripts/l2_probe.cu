// L2 capacity probe (not part of the product): every CTA (one per SM) reads
// the same X-byte buffer `passes` times with L2-only loads, starting at a
// CTA-specific offset. Under ncu, dram__bytes_read ~ X means the buffer stayed
// L2-resident across passes (one shared 126 MB pool); ~ passes * X means it did
// not (e.g. each die keeping its own copy of data both dies' SMs read).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/l2_probe scripts/l2_probe.cu
//   ncu --metrics dram__bytes_read.sum /tmp/l2_probe <MB> <passes>
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

__global__ void probe(const int4* __restrict__ buf, size_t n16, int passes, int* sink) {
    int acc = 0;
    const size_t start = (n16 / gridDim.x) * blockIdx.x;
    for (int p = 0; p < passes; ++p)
        for (size_t i = threadIdx.x; i < n16; i += blockDim.x) {
            size_t j = start + i;
            if (j >= n16) j -= n16;
            const int4 v = __ldcg(buf + j);
            acc ^= v.x ^ v.y ^ v.z ^ v.w;
        }
    if (acc == 0x7fffffff) *sink = acc;
}

int main(int argc, char** argv) {
    const size_t mb = argc > 1 ? atoi(argv[1]) : 64;
    const int passes = argc > 2 ? atoi(argv[2]) : 4;
    const size_t bytes = mb << 20;
    int4* buf;
    int* sink;
    cudaMalloc(&buf, bytes);
    cudaMalloc(&sink, 4);
    cudaMemset(buf, 1, bytes);
    int sms = 0;
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    probe<<<sms, 512>>>(buf, bytes / 16, passes, sink);
    cudaDeviceSynchronize();
    printf("%zu MB x %d passes: %s\n", mb, passes, cudaGetErrorString(cudaGetLastError()));
    return 0;
}
