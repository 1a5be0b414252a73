// Microbenchmark: fixed cost of graph nodes on this GPU (what a small sweep can never beat).
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/graph_floor tools/graph_floor.cu && /tmp/graph_floor
#include <cstdio>
#include <cuda_runtime.h>

__global__ void k_empty(int *p) { if (p && threadIdx.x == 1023) p[0] = 1; }
__global__ void k_smem(int *p) {
    extern __shared__ int s[];
    s[threadIdx.x] = threadIdx.x;
    __syncthreads();
    if (p && s[(threadIdx.x + 1) % blockDim.x] == -1) p[0] = 1;
}

template <class F>
static float per_node_us(cudaStream_t st, int n, F body) {
    cudaGraph_t g;
    cudaGraphExec_t ex;
    cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal);
    for (int i = 0; i < n; ++i) body(st);
    cudaStreamEndCapture(st, &g);
    cudaGraphInstantiate(&ex, g, 0);
    cudaGraphLaunch(ex, st);
    cudaStreamSynchronize(st);
    cudaEvent_t a, b;
    cudaEventCreate(&a);
    cudaEventCreate(&b);
    cudaEventRecord(a, st);
    for (int r = 0; r < 10; ++r) cudaGraphLaunch(ex, st);
    cudaEventRecord(b, st);
    cudaEventSynchronize(b);
    float ms = 0;
    cudaEventElapsedTime(&ms, a, b);
    cudaGraphExecDestroy(ex);
    cudaGraphDestroy(g);
    return 1e3f * ms / (10.f * n);
}

int main() {
    cudaStream_t st;
    cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking);
    int *d;
    cudaMalloc(&d, 1 << 20);
    cudaFuncSetAttribute(k_smem, cudaFuncAttributeMaxDynamicSharedMemorySize, 48 * 1024);
    const int N = 40;
    printf("empty kernel 1x32            : %.2f us/node\n", per_node_us(st, N, [&](cudaStream_t s) { k_empty<<<1, 32, 0, s>>>(d); }));
    printf("empty kernel 148x128         : %.2f us/node\n", per_node_us(st, N, [&](cudaStream_t s) { k_empty<<<148, 128, 0, s>>>(d); }));
    printf("empty kernel 592x128         : %.2f us/node\n", per_node_us(st, N, [&](cudaStream_t s) { k_empty<<<592, 128, 0, s>>>(d); }));
    printf("smem kernel 592x128 45KB     : %.2f us/node\n", per_node_us(st, N, [&](cudaStream_t s) { k_smem<<<592, 128, 45 * 1024, s>>>(d); }));
    printf("smem kernel 868x128 24KB     : %.2f us/node\n", per_node_us(st, N, [&](cudaStream_t s) { k_smem<<<868, 128, 24 * 1024, s>>>(d); }));
    printf("memset 184B                  : %.2f us/node\n", per_node_us(st, N, [&](cudaStream_t s) { cudaMemsetAsync(d, 0xFF, 184, s); }));
    printf("memset 184B + kernel 592x128 : %.2f us/pair\n", per_node_us(st, N, [&](cudaStream_t s) { cudaMemsetAsync(d, 0xFF, 184, s); k_empty<<<592, 128, 0, s>>>(d); }));
    printf("kernel 592 + kernel 148      : %.2f us/pair\n", per_node_us(st, N, [&](cudaStream_t s) { k_empty<<<592, 128, 0, s>>>(d); k_empty<<<148, 256, 0, s>>>(d); }));
    return 0;
}
