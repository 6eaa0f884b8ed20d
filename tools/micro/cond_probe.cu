// Probe: a while-conditional graph node whose body is stream-captured (incl. a fork/join),
// launched (a) as a cached exec graph and (b) inserted into a caller's stream capture.
#include <cstdio>
#include <cuda_runtime.h>
__device__ int g_iter;
__global__ void k_init(int* d, int n, int iters) { if (threadIdx.x == 0 && blockIdx.x == 0) g_iter = iters; }
__global__ void k_work(int* d, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) d[i] += 1;
}
__global__ void k_side(int* d, int n) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x) d[n + i] += 2;
}
__global__ void k_epi(cudaGraphConditionalHandle h) {
    if (threadIdx.x == 0) { int r = --g_iter; cudaGraphSetConditional(h, r > 0 ? 1u : 0u); }
}
__global__ void k_check(int* d, int n, int expect, int* bad) {
    for (int i = blockIdx.x * blockDim.x + threadIdx.x; i < n; i += gridDim.x * blockDim.x)
        if (d[i] != expect / 2 || d[n + i] != expect / 2) atomicAdd(bad, 1);
}
#define CK(x) do { cudaError_t e = (x); if (e != cudaSuccess) { printf("%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); return 1; } } while (0)
static cudaStream_t cs, side; static cudaEvent_t ef, ej;
static int body(cudaStream_t s, cudaGraphConditionalHandle h, int* d, int n) {
    k_work<<<148, 256, 0, s>>>(d, n);
    CK(cudaEventRecord(ef, s)); CK(cudaStreamWaitEvent(side, ef, 0));
    k_side<<<148, 256, 0, side>>>(d, n);
    k_work<<<148, 256, 0, s>>>(d, n);
    CK(cudaEventRecord(ej, side)); CK(cudaStreamWaitEvent(s, ej, 0));
    k_epi<<<1, 32, 0, s>>>(h);
    return 0;
}
static int add_loop(cudaGraph_t g, const cudaGraphNode_t* deps, size_t nd, cudaGraphNode_t* out, int* d, int n) {
    cudaGraphConditionalHandle h;
    CK(cudaGraphConditionalHandleCreate(&h, g, 1, cudaGraphCondAssignDefault));
    cudaGraphNodeParams p = {};
    p.type = cudaGraphNodeTypeConditional;
    p.conditional.handle = h; p.conditional.type = cudaGraphCondTypeWhile; p.conditional.size = 1;
    CK(cudaGraphAddNode(out, g, deps, nd, &p));
    cudaGraph_t b = p.conditional.phGraph_out[0];
    CK(cudaStreamBeginCaptureToGraph(cs, b, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
    if (body(cs, h, d, n)) return 1;
    CK(cudaStreamEndCapture(cs, &b));
    return 0;
}
int main() {
    int n = 1 << 20; int *d, *bad;
    CK(cudaMalloc(&d, 2 * n * 4)); CK(cudaMalloc(&bad, 4));
    cudaStream_t s; CK(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking)); CK(cudaStreamCreateWithFlags(&side, cudaStreamNonBlocking));
    CK(cudaEventCreateWithFlags(&ef, cudaEventDisableTiming)); CK(cudaEventCreateWithFlags(&ej, cudaEventDisableTiming));
    // (a) cached exec graph
    cudaGraph_t g; CK(cudaGraphCreate(&g, 0)); cudaGraphNode_t nd;
    if (add_loop(g, nullptr, 0, &nd, d, n)) return 1;
    cudaGraphExec_t ge; CK(cudaGraphInstantiate(&ge, g, 0));
    for (int iters : {1, 3, 50}) {
        CK(cudaMemsetAsync(d, 0, 2 * n * 4, s)); CK(cudaMemsetAsync(bad, 0, 4, s));
        cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
        k_init<<<1, 32, 0, s>>>(d, n, iters);
        CK(cudaEventRecord(a, s));
        CK(cudaGraphLaunch(ge, s));
        CK(cudaEventRecord(b, s));
        k_check<<<148, 256, 0, s>>>(d, n, 4 * iters, bad);
        int hb = -1; CK(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        float ms; cudaEventElapsedTime(&ms, a, b);
        printf("(a) iters=%d bad=%d %.3f ms (%.2f us/iter, 4 kernels)\n", iters, hb, ms, 1000 * ms / iters);
    }
    // (b) inside a caller's capture
    {
        CK(cudaMemsetAsync(d, 0, 2 * n * 4, s)); CK(cudaMemsetAsync(bad, 0, 4, s)); CK(cudaStreamSynchronize(s));
        CK(cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal));
        k_init<<<1, 32, 0, s>>>(d, n, 7);
        cudaStreamCaptureStatus stt; cudaGraph_t ug; const cudaGraphNode_t* deps; size_t ndeps;
        CK(cudaStreamGetCaptureInfo(s, &stt, nullptr, &ug, &deps, &ndeps));
        cudaGraphNode_t ln;
        if (add_loop(ug, deps, ndeps, &ln, d, n)) return 1;
        CK(cudaStreamUpdateCaptureDependencies(s, &ln, 1, cudaStreamSetCaptureDependencies));
        k_init<<<1, 32, 0, s>>>(d, n, 2);
        cudaGraphNode_t ln2;
        CK(cudaStreamGetCaptureInfo(s, &stt, nullptr, &ug, &deps, &ndeps));
        if (add_loop(ug, deps, ndeps, &ln2, d, n)) return 1;
        CK(cudaStreamUpdateCaptureDependencies(s, &ln2, 1, cudaStreamSetCaptureDependencies));
        cudaGraph_t outg; CK(cudaStreamEndCapture(s, &outg));
        cudaGraphExec_t oe; CK(cudaGraphInstantiate(&oe, outg, 0));
        for (int r = 0; r < 2; ++r) CK(cudaGraphLaunch(oe, s));
        k_check<<<148, 256, 0, s>>>(d, n, 2 * 4 * 9, bad);
        int hb = -1; CK(cudaMemcpyAsync(&hb, bad, 4, cudaMemcpyDeviceToHost, s));
        CK(cudaStreamSynchronize(s));
        printf("(b) captured x2 replays: bad=%d\n", hb);
    }
    return 0;
}
