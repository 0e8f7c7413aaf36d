// Measurement for DESIGN section 9 (leaf apply in a 2-CTA cluster): random 4-byte gathers
// from the peer CTA's shared memory (DSMEM) against the same gathers from local shared
// memory.  One cluster of 2 CTAs per SM pair, 1024 threads per CTA, 128 KB of data per CTA
// (half of a 256 KB uint32 leaf); every thread gathers 64 random elements.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o /tmp/exp_dsmem scripts/exp_dsmem.cu && /tmp/exp_dsmem
#include <cooperative_groups.h>
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>
namespace cg = cooperative_groups;

constexpr int kThreads = 1024, kElems = 32768, kPerThread = 64;

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352du; x ^= x >> 15; x *= 0x846ca68bu; x ^= x >> 16;
  return x;
}

// mode 0: all gathers local; 1: all from the peer CTA; 2: half and half (the leaf's case)
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads)
    gather_kernel(int mode, uint32_t* out, long long* cycles) {
  extern __shared__ uint32_t sdata[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rank = cl.block_rank();
  for (int i = threadIdx.x; i < kElems; i += kThreads) sdata[i] = hash32(i + rank * kElems);
  cl.sync();
  const uint32_t* peer = cl.map_shared_rank(sdata, rank ^ 1);
  uint32_t acc = 0;
  const long long t0 = clock64();
#pragma unroll 8
  for (int k = 0; k < kPerThread; ++k) {
    const uint32_t h = hash32(threadIdx.x * kPerThread + k + blockIdx.x * 977u);
    const uint32_t idx = h & (kElems - 1);
    const bool remote = mode == 1 || (mode == 2 && (h >> 20 & 1));
    acc += remote ? peer[idx] : sdata[idx];
  }
  __syncthreads();
  const long long t1 = clock64();
  cl.sync();
  out[blockIdx.x * kThreads + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

// streaming: every thread reads kElems / kThreads / 4 coalesced 16-byte words, `reps` times
__global__ void __cluster_dims__(2, 1, 1) __launch_bounds__(kThreads)
    stream_kernel(int remote, uint32_t* out, long long* cycles) {
  extern __shared__ uint32_t sdata[];
  cg::cluster_group cl = cg::this_cluster();
  const uint32_t rank = cl.block_rank();
  for (int i = threadIdx.x; i < kElems; i += kThreads) sdata[i] = hash32(i + rank * kElems);
  cl.sync();
  const uint4* src = reinterpret_cast<const uint4*>(remote ? cl.map_shared_rank(sdata, rank ^ 1) : sdata);
  uint32_t acc = 0;
  const long long t0 = clock64();
  for (int rep = 0; rep < 8; ++rep) {
#pragma unroll
    for (int k = 0; k < kElems / 4 / kThreads; ++k) {
      const uint4 v = src[(k * kThreads + threadIdx.x + rep * 32) & (kElems / 4 - 1)];  // (shifted per repetition)
      acc += v.x ^ v.y ^ v.z ^ v.w ^ rep;
    }
    asm volatile("" ::: "memory");  // every repetition loads again
  }
  __syncthreads();
  const long long t1 = clock64();
  cl.sync();
  out[blockIdx.x * kThreads + threadIdx.x] = acc;
  if (threadIdx.x == 0) cycles[blockIdx.x] = t1 - t0;
}

int main() {
  int sms = 0;
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  const int blocks = sms & ~1;
  uint32_t* out;
  long long* cyc;
  cudaMalloc(&out, (size_t)blocks * kThreads * 4);
  cudaMallocManaged(&cyc, blocks * sizeof(long long));
  const size_t smem = (size_t)kElems * 4;
  cudaFuncSetAttribute(gather_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int mode = 0; mode < 3; ++mode) {
    for (int rep = 0; rep < 3; ++rep) {
      gather_kernel<<<blocks, kThreads, smem>>>(mode, out, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; }
    }
    double sum = 0;
    for (int b = 0; b < blocks; ++b) sum += (double)cyc[b];
    const double avg = sum / blocks;
    printf("{\"mode\": \"%s\", \"gathers_per_cta\": %d, \"cycles\": %.0f, \"cycles_per_65536_gathers\": %.0f}\n",
           mode == 0 ? "local smem" : mode == 1 ? "peer smem (DSMEM)" : "half local, half peer",
           kThreads * kPerThread, avg, avg * 65536.0 / (kThreads * kPerThread));
  }
  cudaFuncSetAttribute(stream_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  for (int remote = 0; remote < 2; ++remote) {
    for (int rep = 0; rep < 3; ++rep) {
      stream_kernel<<<blocks, kThreads, smem>>>(remote, out, cyc);
      cudaError_t e = cudaDeviceSynchronize();
      if (e != cudaSuccess) { printf("error: %s\n", cudaGetErrorString(e)); return 1; }
    }
    double sum = 0;
    for (int b = 0; b < blocks; ++b) sum += (double)cyc[b];
    const double avg = sum / blocks, bytes = 8.0 * kElems * 4;
    printf("{\"mode\": \"coalesced 16-byte loads, %s\", \"bytes_per_cta\": %.0f, \"cycles\": %.0f, \"bytes_per_cycle_per_sm\": %.1f}\n",
           remote ? "peer smem (DSMEM)" : "local smem", bytes, avg, bytes / avg);
  }
  return 0;
}
