// Probe: does a launch with BOTH cudaLaunchAttributeCooperative and programmatic stream
// serialization (PDL) work on sm_100a, eagerly and under stream capture?
#include <cstdio>
#include <cuda_runtime.h>
__global__ void k(int* out) {
    asm volatile("griddepcontrol.wait;" ::: "memory");
    if (threadIdx.x == 0) atomicAdd(out, 1);
    asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
}
static cudaError_t launch(cudaStream_t s, int* out, bool coop, bool pdl, int grid) {
    cudaLaunchConfig_t cfg{};
    cfg.gridDim = grid; cfg.blockDim = 288; cfg.stream = s;
    cudaLaunchAttribute a[2]; int n = 0;
    if (coop) { a[n].id = cudaLaunchAttributeCooperative; a[n].val.cooperative = 1; ++n; }
    if (pdl) { a[n].id = cudaLaunchAttributeProgrammaticStreamSerialization; a[n].val.programmaticStreamSerializationAllowed = 1; ++n; }
    cfg.attrs = a; cfg.numAttrs = n;
    return cudaLaunchKernelEx(&cfg, k, out);
}
int main() {
    int* out; cudaMalloc(&out, 4); cudaMemset(out, 0, 4);
    cudaStream_t s; cudaStreamCreate(&s);
    int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
    int occ = 0; cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k, 288, 0);
    printf("sms %d occ %d\n", sms, occ);
    for (int coop = 0; coop < 2; ++coop) for (int pdl = 0; pdl < 2; ++pdl) {
        cudaError_t e1 = launch(s, out, coop, pdl, 2 * sms);
        cudaError_t e2 = launch(s, out, coop, pdl, 2 * sms);
        cudaError_t e3 = cudaStreamSynchronize(s);
        printf("eager coop=%d pdl=%d: %s %s %s\n", coop, pdl, cudaGetErrorString(e1), cudaGetErrorString(e2), cudaGetErrorString(e3));
        cudaGetLastError();
        cudaGraph_t g; cudaGraphExec_t ge;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeGlobal);
        e1 = launch(s, out, coop, pdl, 2 * sms);
        e2 = launch(s, out, coop, pdl, 2 * sms);
        cudaError_t e4 = cudaStreamEndCapture(s, &g);
        cudaError_t e5 = e4 == cudaSuccess ? cudaGraphInstantiate(&ge, g, 0) : e4;
        cudaError_t e6 = e5 == cudaSuccess ? cudaGraphLaunch(ge, s) : e5;
        e3 = cudaStreamSynchronize(s);
        printf("graph coop=%d pdl=%d: %s %s end %s inst %s launch %s sync %s\n", coop, pdl, cudaGetErrorString(e1),
               cudaGetErrorString(e2), cudaGetErrorString(e4), cudaGetErrorString(e5), cudaGetErrorString(e6), cudaGetErrorString(e3));
        cudaGetLastError();
    }
    // too large a cooperative grid must be rejected, not hang
    cudaError_t e = launch(s, out, true, true, 64 * sms);
    printf("coop oversize: %s\n", cudaGetErrorString(e));
    int h; cudaMemcpy(&h, out, 4, cudaMemcpyDeviceToHost); printf("count %d\n", h);
    return 0;
}
