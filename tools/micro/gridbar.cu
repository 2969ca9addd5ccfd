// Grid-barrier latency on B200: 148 co-resident CTAs x 448 threads (cooperative launch), NB back-to-back barriers,
// optionally after STORES bytes of global stores per CTA (the release must wait for them).  Variants:
//  0  the persistent kernel's: red.release.gpu.add + ld.acquire.gpu polling by thread 0
//  1  fence.acq_rel.gpu + red.relaxed.gpu + ld.relaxed.gpu polling, one fence.acq_rel after the wait
//  2  as 0, polling with __nanosleep(32) back-off
//  3  two-level: CTAs of a cluster pair (barrier.cluster) -> one arrival per pair on the counter -> cluster barrier
//  4  as 0 but the counter line read by polls is a separate flag written by the last arriver (atom.add.acq_rel)
// nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gridbar gridbar.cu && ./gridbar
#include <cooperative_groups.h>
#include <cstdio>
#include <cuda_runtime.h>

__device__ __forceinline__ unsigned ld_acq(const unsigned* p) {
  unsigned v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned ld_rlx(const unsigned* p) {
  unsigned v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void red_rel(unsigned* p, unsigned v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void red_rlx(unsigned* p, unsigned v) {
  asm volatile("red.relaxed.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ unsigned atom_acqrel(unsigned* p, unsigned v) {
  unsigned o;
  asm volatile("atom.acq_rel.gpu.global.add.u32 %0, [%1], %2;" : "=r"(o) : "l"(p), "r"(v) : "memory");
  return o;
}
__device__ __forceinline__ void st_rel(unsigned* p, unsigned v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ void cl_arrive() { asm volatile("barrier.cluster.arrive.release.aligned;" ::: "memory"); }
__device__ __forceinline__ void cl_wait() { asm volatile("barrier.cluster.wait.acquire.aligned;" ::: "memory"); }

template <int V>
__global__ void __launch_bounds__(448, 1) kbar(unsigned* cnt, unsigned* flag, float* junk, int nb, int stores,
                                               long long* out) {
  const int tid = threadIdx.x;
  unsigned gen = 0;
  long long t0 = 0;
  for (int i = 0; i < nb; ++i) {
    if (i == 8) t0 = clock64();
    // the phase's stores (16-byte, this CTA's own region)
    float4* dst = reinterpret_cast<float4*>(junk) + (size_t)blockIdx.x * (stores / 16);
    for (int e = tid; e < stores / 16; e += blockDim.x) dst[e] = make_float4(i, e, 0, 1);
    ++gen;
    if (V == 0 || V == 2) {
      __syncthreads();
      if (tid == 0) {
        red_rel(cnt, 1u);
        while ((int)(ld_acq(cnt) - gen * gridDim.x) < 0) {
          if (V == 2) __nanosleep(32);
        }
      }
      __syncthreads();
    } else if (V == 1) {
      __syncthreads();
      if (tid == 0) {
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
        red_rlx(cnt, 1u);
        while ((int)(ld_rlx(cnt) - gen * gridDim.x) < 0) {
        }
        asm volatile("fence.acq_rel.gpu;" ::: "memory");
      }
      __syncthreads();
    } else if (V == 3) {
      cl_arrive();
      cl_wait();
      const unsigned pairs = gridDim.x / 2;
      if (tid == 0 && (blockIdx.x & 1) == 0) {
        red_rel(cnt, 1u);
        while ((int)(ld_acq(cnt) - gen * pairs) < 0) {
        }
      }
      cl_arrive();
      cl_wait();
    } else if (V == 4) {
      __syncthreads();
      if (tid == 0) {
        const unsigned o = atom_acqrel(cnt, 1u);
        if (o == gen * gridDim.x - 1) st_rel(flag, gen);
        else
          while ((int)(ld_acq(flag) - gen) < 0) {
          }
      }
      __syncthreads();
    }
  }
  if (tid == 0) out[blockIdx.x] = clock64() - t0;
}

template <int V>
float run(int nb, int stores, int cluster) {
  unsigned *cnt, *flag;
  float* junk;
  long long* out;
  cudaMalloc(&cnt, 256);
  cudaMalloc(&flag, 256);
  cudaMalloc(&junk, (size_t)148 * (stores + 16));
  cudaMalloc(&out, 148 * 8);
  cudaMemset(cnt, 0, 256);
  cudaMemset(flag, 0, 256);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(148);
  cfg.blockDim = dim3(448);
  cudaLaunchAttribute at[2];
  int na = 0;
  at[na].id = cudaLaunchAttributeCooperative;
  at[na++].val.cooperative = 1;
  if (cluster > 1) {
    at[na].id = cudaLaunchAttributeClusterDimension;
    at[na].val.clusterDim.x = cluster;
    at[na].val.clusterDim.y = 1;
    at[na++].val.clusterDim.z = 1;
  }
  cfg.attrs = at;
  cfg.numAttrs = na;
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  cudaEventRecord(e0);
  cudaError_t err = cudaLaunchKernelEx(&cfg, kbar<V>, cnt, flag, junk, nb, stores, out);
  cudaEventRecord(e1);
  cudaError_t e2 = cudaDeviceSynchronize();
  float ms = 0;
  cudaEventElapsedTime(&ms, e0, e1);
  if (err != cudaSuccess || e2 != cudaSuccess) printf("V%d err %s %s\n", V, cudaGetErrorString(err), cudaGetErrorString(e2));
  cudaFree(cnt);
  cudaFree(flag);
  cudaFree(junk);
  cudaFree(out);
  return ms * 1e3f / nb;
}

int main() {
  const int nb = 4000;
  for (int stores : {0, 16384}) {
    for (int rep = 0; rep < 2; ++rep) {
      printf("stores %5d B/CTA: V0 %.3f  V1 %.3f  V2 %.3f  V3 %.3f  V4 %.3f us/barrier\n", stores, run<0>(nb, stores, 1),
             run<1>(nb, stores, 1), run<2>(nb, stores, 1), run<3>(nb, stores, 2), run<4>(nb, stores, 1));
    }
  }
  return 0;
}
