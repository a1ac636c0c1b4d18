// Can a captured cudaMemcpyAsync node's host end be re-pointed in an instantiated graph?
#include <cstdio>
#include <cuda_runtime.h>
int main() {
    cudaStream_t s; cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
    double *h1, *h2, *d;
    cudaHostAlloc(&h1, 1 << 20, 0); cudaHostAlloc(&h2, 1 << 20, 0); cudaMalloc(&d, 1 << 20);
    cudaGraph_t g; cudaGraphExec_t e;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    cudaMemcpyAsync(h1, d, 1 << 20, cudaMemcpyDeviceToHost, s);
    cudaStreamEndCapture(s, &g);
    size_t n = 0; cudaGraphGetNodes(g, nullptr, &n);
    cudaGraphNode_t nd; cudaGraphGetNodes(g, &nd, &n);
    cudaMemcpy3DParms p{}; cudaError_t r = cudaGraphMemcpyNodeGetParams(nd, &p);
    printf("get %s kind %d src %p dst %p extent %zu %zu %zu srcpitch %zu\n", cudaGetErrorString(r), (int)p.kind,
           p.srcPtr.ptr, p.dstPtr.ptr, p.extent.width, p.extent.height, p.extent.depth, p.srcPtr.pitch);
    printf("inst %s\n", cudaGetErrorString(cudaGraphInstantiate(&e, g, 0)));
    cudaMemcpy3DParms q = p; q.dstPtr.ptr = h2;
    printf("set3D %s\n", cudaGetErrorString(cudaGraphExecMemcpyNodeSetParams(e, nd, &q)));
    cudaGetLastError();
    printf("set1D %s\n", cudaGetErrorString(cudaGraphExecMemcpyNodeSetParams1D(e, nd, h2, d, 1 << 20, cudaMemcpyDeviceToHost)));
    cudaGetLastError();
    printf("set1D default %s\n", cudaGetErrorString(cudaGraphExecMemcpyNodeSetParams1D(e, nd, h2, d, 1 << 20, cudaMemcpyDefault)));
    cudaGetLastError();
    cudaMemcpy3DParms z = p; z.dstPtr.ptr = h2; z.kind = cudaMemcpyDefault;
    printf("set3D default %s\n", cudaGetErrorString(cudaGraphExecMemcpyNodeSetParams(e, nd, &z)));
    cudaGetLastError();
    // node-level update then re-instantiate-free update path
    printf("graph-node set %s\n", cudaGetErrorString(cudaGraphMemcpyNodeSetParams(nd, &q)));
    cudaGraphExecUpdateResultInfo info;
    printf("exec update %s\n", cudaGetErrorString(cudaGraphExecUpdate(e, g, &info)));
    printf("launch %s sync %s\n", cudaGetErrorString(cudaGraphLaunch(e, s)), cudaGetErrorString(cudaStreamSynchronize(s)));
    // registered (cudaHostRegister) host memory as the new end
    double* h3 = (double*)malloc(1 << 20);
    printf("register %s\n", cudaGetErrorString(cudaHostRegister(h3, 1 << 20, 0)));
    cudaMemcpy3DParms w = p; w.dstPtr.ptr = h3;
    printf("set3D registered %s\n", cudaGetErrorString(cudaGraphExecMemcpyNodeSetParams(e, nd, &w)));
    cudaGetLastError();
    // offset into a pinned block
    cudaMemcpy3DParms o = p; o.dstPtr.ptr = (char*)h2 + 4096;
    printf("set3D offset %s\n", cudaGetErrorString(cudaGraphExecMemcpyNodeSetParams(e, nd, &o)));
    cudaGetLastError();
    // interior pointer, in range: a second graph copying half a block
    {
        cudaGraph_t g2; cudaGraphExec_t e2;
        cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        cudaMemcpyAsync(h1, d, 1 << 19, cudaMemcpyDeviceToHost, s);
        cudaStreamEndCapture(s, &g2);
        size_t n2 = 0; cudaGraphGetNodes(g2, nullptr, &n2);
        cudaGraphNode_t nd2; cudaGraphGetNodes(g2, &nd2, &n2);
        cudaMemcpy3DParms p2{}; cudaGraphMemcpyNodeGetParams(nd2, &p2);
        cudaGraphInstantiate(&e2, g2, 0);
        cudaMemcpy3DParms i2 = p2; i2.dstPtr.ptr = (char*)h2 + 4096;
        printf("set3D interior in-range %s\n", cudaGetErrorString(cudaGraphExecMemcpyNodeSetParams(e2, nd2, &i2)));
        cudaGetLastError();
        cudaMemcpy3DParms i3 = p2; i3.dstPtr.ptr = (char*)h1 + 4096;
        printf("set3D interior same block %s\n", cudaGetErrorString(cudaGraphExecMemcpyNodeSetParams(e2, nd2, &i3)));
        cudaGetLastError();
    }
    // smaller host allocation than the copy? (same size copy into a fresh 1 MB block)
    double* h4; cudaHostAlloc(&h4, 1 << 20, cudaHostAllocPortable | cudaHostAllocMapped);
    cudaMemcpy3DParms m = p; m.dstPtr.ptr = h4;
    printf("set3D mapped %s\n", cudaGetErrorString(cudaGraphExecMemcpyNodeSetParams(e, nd, &m)));
    cudaGetLastError();
    return 0;
}
