// Random-gather microbenchmark ("a random-16 B-gather microbenchmark peak measured
// on the box, so the binding level is visible").  Not part of the product; built and run by
// tools/gather_peak.sh on the GPU box.
//
// For working sets from 64 KiB (L1-resident) to 2 GiB (HBM), every lane issues independent
// loads from hashed pseudo-random addresses (no index traffic) and reports
//   * useful GB/s     = loads x access width / time
//   * loads/s (G/s)   = the gather-rate ceiling a walk step can hope for at that level
// for 16 B (the walk's float4 neighbour record) and 32 B (the 256-bit pair loads) accesses, and,
// as the best case of a coherent warp, a warp-uniform random line (lanes read consecutive 16 B).
// A dependent pointer chase (one warp per SM, random cyclic permutation) gives the latency.
#include <cuda_runtime.h>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <vector>
#include <algorithm>
#include <random>

#define CK(x) do { cudaError_t e_ = (x); if (e_ != cudaSuccess) { \
  fprintf(stderr, "%s:%d %s\n", __FILE__, __LINE__, cudaGetErrorString(e_)); exit(1); } } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t x) {
  x ^= x >> 16; x *= 0x7feb352dU; x ^= x >> 15; x *= 0x846ca68bU; x ^= x >> 16; return x;
}

struct alignas(32) v8 { float a[8]; };

__device__ __forceinline__ void ld32(const void *p, float4 &a, float4 &b) {
  asm volatile("ld.global.nc.v8.f32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];"
               : "=f"(a.x), "=f"(a.y), "=f"(a.z), "=f"(a.w), "=f"(b.x), "=f"(b.y), "=f"(b.z), "=f"(b.w)
               : "l"(p));
}

// MODE 0: per-lane random 16 B; 1: per-lane random 32 B; 2: warp-uniform random 512 B line group.
template <int MODE, int ILP>
__global__ void __launch_bounds__(256) k_gather(const float4 *__restrict__ buf, uint32_t mask16,
                                                int iters, uint32_t seed, float *__restrict__ sink) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t lane = threadIdx.x & 31;
  float acc = 0.f;
  for (int it = 0; it < iters; ++it) {
    float4 v[ILP];
    float4 w[ILP];
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      uint32_t h;
      if (MODE == 2) h = ((hash32((tid >> 5) * 0x9e3779b9U + (it * ILP + k) * 0x85ebca6bU + seed) << 5) + lane) & mask16;
      else h = hash32(tid * 0x9e3779b9U + (it * ILP + k) * 0x85ebca6bU + seed) & mask16;
      if (MODE == 1) {
        ld32(buf + (h & ~1u), v[k], w[k]);
      } else {
        v[k] = __ldg(buf + h);
      }
    }
#pragma unroll
    for (int k = 0; k < ILP; ++k) {
      acc += v[k].x + v[k].y + v[k].z + v[k].w;
      if (MODE == 1) acc += w[k].x + w[k].y + w[k].z + w[k].w;
    }
  }
  if (acc == 1234.5f) sink[tid] = acc;
}

__global__ void k_chase(const uint32_t *__restrict__ next, uint32_t slots, int hops,
                        uint32_t *__restrict__ out) {
  uint32_t p = (uint32_t)(((uint64_t)blockIdx.x * 0x9e3779b9u) % slots) * 16u;  // one per block
  for (int i = 0; i < hops; ++i) p = __ldcg(next + p);  // bypass L1: L2 / HBM latency
  if (threadIdx.x == 0) out[blockIdx.x] = p;
}

__global__ void k_fill(float4 *buf, size_t n) {
  size_t i = blockIdx.x * (size_t)blockDim.x + threadIdx.x;
  for (; i < n; i += (size_t)gridDim.x * blockDim.x) buf[i] = make_float4(1e-9f, 0.f, 0.f, 0.f);
}

template <int MODE>
static void run(const float4 *buf, size_t bytes, int sms, float *sink, const char *label) {
  constexpr int ILP = 8;
  uint32_t mask16 = (uint32_t)(bytes / 16 - 1);
  int blocks = sms * 8, threads = 256;
  int iters = 64;
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  k_gather<MODE, ILP><<<blocks, threads>>>(buf, mask16, iters, 1, sink);
  CK(cudaDeviceSynchronize());
  float best = 1e30f;
  for (int r = 0; r < 5; ++r) {
    CK(cudaEventRecord(e0));
    k_gather<MODE, ILP><<<blocks, threads>>>(buf, mask16, iters, 2 + r, sink);
    CK(cudaEventRecord(e1));
    CK(cudaEventSynchronize(e1));
    float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
    best = std::min(best, ms);
  }
  double loads = (double)blocks * threads * iters * ILP;
  double width = MODE == 1 ? 32.0 : 16.0;
  printf("{\"kind\": \"gather\", \"access\": \"%s\", \"working_set_bytes\": %zu, \"ms\": %.4f, "
         "\"gloads_per_s\": %.2f, \"useful_GBps\": %.1f}\n",
         label, bytes, best, loads / best / 1e6, loads * width / best / 1e6);
  CK(cudaEventDestroy(e0)); CK(cudaEventDestroy(e1));
}

static void chase(size_t bytes, int sms) {
  size_t n = bytes / 4;
  // Sattolo: one random cycle over n/16 slots spaced a 64 B line apart (defeats the line reuse)
  size_t slots = n / 16;
  std::vector<uint32_t> perm(slots);
  for (size_t i = 0; i < slots; ++i) perm[i] = (uint32_t)i;
  std::mt19937_64 rng(7);
  for (size_t i = slots - 1; i > 0; --i) {
    size_t j = rng() % i;
    std::swap(perm[i], perm[j]);
  }
  std::vector<uint32_t> next(n, 0);
  for (size_t i = 0; i < slots; ++i) next[i * 16] = perm[i] * 16;
  uint32_t *d_next, *d_out;
  CK(cudaMalloc(&d_next, n * 4)); CK(cudaMalloc(&d_out, sms * 4));
  CK(cudaMemcpy(d_next, next.data(), n * 4, cudaMemcpyHostToDevice));
  int hops = 20000;
  k_chase<<<sms, 32>>>(d_next, (uint32_t)slots, 1000, d_out);
  CK(cudaDeviceSynchronize());
  cudaEvent_t e0, e1;
  CK(cudaEventCreate(&e0)); CK(cudaEventCreate(&e1));
  CK(cudaEventRecord(e0));
  k_chase<<<sms, 32>>>(d_next, (uint32_t)slots, hops, d_out);
  CK(cudaEventRecord(e1));
  CK(cudaEventSynchronize(e1));
  float ms; CK(cudaEventElapsedTime(&ms, e0, e1));
  printf("{\"kind\": \"chase\", \"working_set_bytes\": %zu, \"ns_per_hop\": %.1f}\n", bytes,
         ms * 1e6 / hops);
  CK(cudaFree(d_next)); CK(cudaFree(d_out));
}

int main() {
  int dev = 0, sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev));
  size_t maxb = (size_t)2 << 30;
  float4 *buf; float *sink;
  CK(cudaMalloc(&buf, maxb));
  CK(cudaMalloc(&sink, (size_t)sms * 8 * 256 * 4));
  k_fill<<<sms * 8, 256>>>(buf, maxb / 16);
  CK(cudaDeviceSynchronize());
  std::vector<size_t> sizes;
  for (size_t b = (size_t)64 << 10; b < maxb; b <<= 2) sizes.push_back(b);
  sizes.push_back(maxb);
  for (size_t b : sizes) {
    run<0>(buf, b, sms, sink, "lane16");
    run<1>(buf, b, sms, sink, "lane32");
    run<2>(buf, b, sms, sink, "warp512");
  }
  chase((size_t)32 << 20, sms);
  chase((size_t)1 << 30, sms);
  CK(cudaFree(buf)); CK(cudaFree(sink));
  return 0;
}
