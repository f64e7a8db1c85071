// Dev probe: launch overhead per kernel on B200 for the shapes of the small-n single launch:
// back-to-back launches of an (almost) empty kernel with 148 CTAs x 256 threads and 16 KB of
// dynamic shared memory -- cooperative launch (grid.sync once) vs normal launch vs a
// 16-CTA cluster launch -- directly and captured in a CUDA graph; us per launch.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/launch_probe tools/probe/launch_probe.cu
#include <cooperative_groups.h>
#include <cstdio>
namespace cg = cooperative_groups;

__global__ void k_coop(int* p) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  cg::this_grid().sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += sm[5];
}
__global__ void k_plain(int* p) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  __syncthreads();
  if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += sm[5];
}
__global__ void k_cluster(int* p) {
  extern __shared__ int sm[];
  sm[threadIdx.x] = threadIdx.x;
  cg::this_cluster().sync();
  if (threadIdx.x == 0 && blockIdx.x == 0) p[0] += sm[5];
}

template <class F>
float time_us(F launch, cudaStream_t s, int reps, bool graph) {
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  cudaGraphExec_t ge = nullptr;
  if (graph) {
    cudaGraph_t g;
    cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
    for (int i = 0; i < reps; ++i) launch();
    cudaStreamEndCapture(s, &g);
    cudaGraphInstantiate(&ge, g, 0);
    cudaGraphLaunch(ge, s);
  } else {
    for (int i = 0; i < reps; ++i) launch();
  }
  cudaStreamSynchronize(s);
  float best = 1e30f;
  for (int t = 0; t < 5; ++t) {
    cudaEventRecord(a, s);
    if (graph) cudaGraphLaunch(ge, s);
    else for (int i = 0; i < reps; ++i) launch();
    cudaEventRecord(b, s);
    cudaEventSynchronize(b);
    float ms;
    cudaEventElapsedTime(&ms, a, b);
    best = ms * 1e3f / reps < best ? ms * 1e3f / reps : best;
  }
  return best;
}

int main() {
  int* p;
  cudaMalloc(&p, 4);
  cudaStream_t s;
  cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking);
  const size_t smem = 16384;
  const int reps = 200;
  void* args[] = {&p};
  auto coop = [&] { cudaLaunchCooperativeKernel((void*)k_coop, dim3(148), dim3(256), args, smem, s); };
  auto plain = [&] { k_plain<<<148, 256, smem, s>>>(p); };
  auto plain16 = [&] { k_plain<<<16, 256, smem, s>>>(p); };
  cudaFuncSetAttribute(k_cluster, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  auto cluster16 = [&] {
    cudaLaunchConfig_t cfg = {};
    cfg.gridDim = dim3(16);
    cfg.blockDim = dim3(256);
    cfg.dynamicSmemBytes = smem;
    cfg.stream = s;
    cudaLaunchAttribute at[1];
    at[0].id = cudaLaunchAttributeClusterDimension;
    at[0].val.clusterDim.x = 16;
    at[0].val.clusterDim.y = 1;
    at[0].val.clusterDim.z = 1;
    cfg.attrs = at;
    cfg.numAttrs = 1;
    cudaLaunchKernelEx(&cfg, k_cluster, p);
  };
  for (int gph = 0; gph < 2; ++gph) {
    printf("{\"graph\": %d, \"coop148_us\": %.2f, \"plain148_us\": %.2f, \"plain16_us\": %.2f, \"cluster16_us\": %.2f, \"err\": \"%s\"}\n",
           gph, time_us(coop, s, reps, gph), time_us(plain, s, reps, gph), time_us(plain16, s, reps, gph),
           time_us(cluster16, s, reps, gph), cudaGetErrorString(cudaGetLastError()));
  }
  return 0;
}
