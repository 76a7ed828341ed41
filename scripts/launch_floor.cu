// Launch-latency floor of a one-wave round on B200 (development probe for small layouts).
//
// Times CUDA graphs of 100 back-to-back launches, with and without programmatic dependent
// launch (PDL), of kernels shaped like the ResNet-20 fused round (284 CTAs x 256 threads,
// 2 CTAs/SM by register budget):
//   empty   : nothing
//   pdl     : griddepcontrol.wait + launch_dependents only
//   stream  : + per warp one chunk of the round's traffic (g 512 B, r 1 KB, W 1 KB in;
//             r' 1 KB, W' 1 KB, loc 512 B out), L2-resident buffers
//   stream+red : + one fp64 atomic per CTA to one address (the grad-norm partial)
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o launch_floor scripts/launch_floor.cu
//   ./launch_floor [ctas=284]
#include <cstdio>
#include <cstdlib>
#include <cuda_runtime.h>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { printf("%s: %s\n", #x, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ void pdl_wait() { asm volatile("griddepcontrol.wait;" ::: "memory"); }
__device__ __forceinline__ void pdl_trigger() { asm volatile("griddepcontrol.launch_dependents;" :::); }

struct Bufs {
    const float* g;
    const double* r_in;
    double* r_out;
    double* W;
    float* loc;
    double* acc;
};

// the engine's access flavours: ld.global.nc.L1::no_allocate (128/256-bit) and st.global.cs
__device__ __forceinline__ float4 ld_nc(const float* p) {
    float4 v;
    asm("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];" : "=f"(v.x), "=f"(v.y), "=f"(v.z), "=f"(v.w) : "l"(p));
    return v;
}
struct d4 { double x, y, z, w; };
__device__ __forceinline__ d4 ld_nc(const double* p) {
    d4 v;
    asm("ld.global.nc.L1::no_allocate.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v.x), "=d"(v.y), "=d"(v.z), "=d"(v.w) : "l"(p));
    return v;
}
__device__ __forceinline__ void st_cs(double* p, d4 v) {
    asm volatile("st.global.cs.v4.f64 [%0], {%1,%2,%3,%4};" ::"l"(p), "d"(v.x), "d"(v.y), "d"(v.z), "d"(v.w));
}
__device__ __forceinline__ void st_cs(float* p, float4 v) {
    asm volatile("st.global.cs.v4.f32 [%0], {%1,%2,%3,%4};" ::"l"(p), "f"(v.x), "f"(v.y), "f"(v.z), "f"(v.w));
}

template <int MODE>
__global__ void __launch_bounds__(256, 2) k_probe(Bufs b) {
    if (MODE >= 4) {  // the same traffic with the engine's access flavours
        pdl_wait();
        pdl_trigger();
        const int lane = threadIdx.x & 31;
        const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
        const long long e = w * 128 + 4 * lane;
        const float4 g = ld_nc(b.g + e);
        const d4 r = ld_nc(b.r_in + e);
        d4 wv = ld_nc(b.W + e);
        wv.x -= 0.1 * g.x; wv.y -= 0.1 * g.y; wv.z -= 0.1 * g.z; wv.w -= 0.1 * g.w;
        st_cs(b.r_out + e, d4{r.x + g.x, r.y + g.y, r.z + g.z, r.w + g.w});
        st_cs(b.W + e, wv);
        st_cs(b.loc + e, make_float4(static_cast<float>(wv.x), static_cast<float>(wv.y), static_cast<float>(wv.z),
                                     static_cast<float>(wv.w)));
        return;
    }
    if (MODE >= 1) {
        pdl_wait();
        pdl_trigger();
    }
    if (MODE >= 2) {
        const int lane = threadIdx.x & 31;
        const long long w = (static_cast<long long>(blockIdx.x) * blockDim.x + threadIdx.x) >> 5;
        const long long e = w * 128 + 4 * lane;
        const float4 g = *reinterpret_cast<const float4*>(b.g + e);
        const double2 r0 = *reinterpret_cast<const double2*>(b.r_in + e);
        const double2 r1 = *reinterpret_cast<const double2*>(b.r_in + e + 2);
        double2 w0 = *reinterpret_cast<const double2*>(b.W + e);
        double2 w1 = *reinterpret_cast<const double2*>(b.W + e + 2);
        w0.x -= 0.1 * g.x; w0.y -= 0.1 * g.y; w1.x -= 0.1 * g.z; w1.y -= 0.1 * g.w;
        *reinterpret_cast<double2*>(b.r_out + e) = make_double2(r0.x + g.x, r0.y + g.y);
        *reinterpret_cast<double2*>(b.r_out + e + 2) = make_double2(r1.x + g.z, r1.y + g.w);
        *reinterpret_cast<double2*>(b.W + e) = w0;
        *reinterpret_cast<double2*>(b.W + e + 2) = w1;
        *reinterpret_cast<float4*>(b.loc + e) =
            make_float4(static_cast<float>(w0.x), static_cast<float>(w0.y), static_cast<float>(w1.x), static_cast<float>(w1.y));
        if (MODE >= 3) {
            __syncthreads();
            if (threadIdx.x == 0) atomicAdd(b.acc, 1.0);
        }
    }
}

template <int MODE>
float time_graph(int ctas, bool pdl, const Bufs& b, cudaStream_t st) {
    cudaGraph_t g;
    cudaGraphExec_t ge;
    CK(cudaStreamBeginCapture(st, cudaStreamCaptureModeGlobal));
    for (int i = 0; i < 100; ++i) {
        cudaLaunchConfig_t cfg = {};
        cfg.gridDim = dim3(ctas);
        cfg.blockDim = dim3(256);
        cfg.stream = st;
        cudaLaunchAttribute attr[1];
        attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
        attr[0].val.programmaticStreamSerializationAllowed = 1;
        cfg.attrs = attr;
        cfg.numAttrs = pdl ? 1 : 0;
        CK(cudaLaunchKernelEx(&cfg, k_probe<MODE>, b));
    }
    CK(cudaStreamEndCapture(st, &g));
    CK(cudaGraphInstantiate(&ge, g, 0));
    for (int i = 0; i < 5; ++i) CK(cudaGraphLaunch(ge, st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    CK(cudaStreamSynchronize(st));
    CK(cudaEventRecord(e0, st));
    for (int i = 0; i < 50; ++i) CK(cudaGraphLaunch(ge, st));
    CK(cudaEventRecord(e1, st));
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    CK(cudaEventElapsedTime(&ms, e0, e1));
    CK(cudaGraphExecDestroy(ge));
    CK(cudaGraphDestroy(g));
    return 1e3f * ms / 5000.f;  // us per launch
}

int main(int argc, char** argv) {
    const int ctas = argc > 1 ? atoi(argv[1]) : 284;
    const long long n = static_cast<long long>(ctas) * 8 * 128;
    Bufs b;
    CK(cudaMalloc(const_cast<float**>(&b.g), n * 4));
    CK(cudaMalloc(const_cast<double**>(&b.r_in), n * 8));
    CK(cudaMalloc(&b.r_out, n * 8));
    CK(cudaMalloc(&b.W, n * 8));
    CK(cudaMalloc(&b.loc, n * 4));
    CK(cudaMalloc(&b.acc, 8));
    CK(cudaMemset(const_cast<float*>(b.g), 0, n * 4));
    CK(cudaMemset(const_cast<double*>(b.r_in), 0, n * 8));
    CK(cudaMemset(b.W, 0, n * 8));
    cudaStream_t st;
    CK(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking));
    printf("{\"ctas\": %d, \"elements\": %lld", ctas, n);
    const char* names[5] = {"empty", "pdl", "stream", "stream_red", "stream_nc_cs"};
    for (int pdl = 0; pdl < 2; ++pdl) {
        float t[5] = {time_graph<0>(ctas, pdl, b, st), time_graph<1>(ctas, pdl, b, st), time_graph<2>(ctas, pdl, b, st),
                      time_graph<3>(ctas, pdl, b, st), time_graph<4>(ctas, pdl, b, st)};
        for (int m = 0; m < 5; ++m) printf(", \"%s%s_us\": %.3f", names[m], pdl ? "_pdlattr" : "", t[m]);
    }
    printf("}\n");
    return 0;
}
