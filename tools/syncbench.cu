// syncbench.cu — latency constants of the Stream-K fixup's synchronisation on B200.
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o tools/syncbench tools/syncbench.cu && tools/syncbench
// (1) what __nanosleep(t) really sleeps; (2) ld.acquire.gpu round trip on an L2-resident
// flag; (3) one-way flag visibility between two CTAs (ping-pong / 2) for several poll loops;
// (4) store S bytes + fence.acq_rel.gpu + st.release, one CTA alone and all 148 at once;
// (5) the fixup pattern at full chip: every CTA stores a partial, releases its flag and waits
// for a neighbour's flag — time from the neighbour's release to the observation.
#include <cuda_runtime.h>

#include <algorithm>
#include <cstdint>
#include <cstdio>
#include <vector>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      printf("CUDA error %s at %s:%d\n", cudaGetErrorString(e), __FILE__, __LINE__);  \
      return 1;                                                                        \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_release(uint32_t* p, uint32_t v) {
  asm volatile("st.release.gpu.global.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}
__device__ __forceinline__ uint64_t gtimer() {
  uint64_t t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

// (1) nanosleep durations, (2) acquire-load round trip
__global__ void k_sleep(long long* out, const uint32_t* flag) {
  if (threadIdx.x != 0) return;
  const int ts[6] = {0, 32, 100, 256, 1000, 4000};
  for (int i = 0; i < 6; ++i) {
    long long t0 = clock64();
    for (int r = 0; r < 64; ++r) __nanosleep(ts[i]);
    out[i] = (clock64() - t0) / 64;
  }
  uint32_t acc = 0;
  long long t0 = clock64();
  for (int r = 0; r < 64; ++r) acc += ld_acquire(flag + (acc & 0));
  out[6] = (clock64() - t0) / 64;
  t0 = clock64();
  for (int r = 0; r < 64; ++r) acc += ld_relaxed(flag + (acc & 0));
  out[7] = (clock64() - t0) / 64 + (acc == 12345 ? 1 : 0);
  // %globaltimer: cycles per read, and the distinct values seen over ~20 us (update granularity)
  uint64_t g0 = gtimer(), gl = g0, steps = 0;
  t0 = clock64();
  for (int r = 0; r < 64; ++r) {
    const uint64_t g = gtimer();
    if (g != gl) ++steps;
    gl = g;
  }
  out[8] = (clock64() - t0) / 64;
  t0 = clock64();
  uint64_t changes = 0, last = gtimer(), first = last;
  while (clock64() - t0 < 40000) {
    const uint64_t g = gtimer();
    if (g != last) ++changes;
    last = g;
  }
  out[9] = (long long)changes;
  out[10] = (long long)(last - first);
  out[11] = (long long)steps;
}

// (3) ping-pong between CTA 0 and CTA 1 (mode: 0 spin, 1 nanosleep(32), 2 nanosleep(100))
__global__ void k_pingpong(uint32_t* f, int iters, int mode, long long* out) {
  if (threadIdx.x != 0) return;
  uint32_t* mine = f + 32 * blockIdx.x;
  const uint32_t* other = f + 32 * (1 - blockIdx.x);
  long long t0 = clock64();
  for (int i = 1; i <= iters; ++i) {
    if (blockIdx.x == 0) {
      st_release(mine, i);
      while (ld_acquire(other) != (uint32_t)i) {
        if (mode == 1) __nanosleep(32);
        if (mode == 2) __nanosleep(100);
      }
    } else {
      while (ld_acquire(other) != (uint32_t)i) {
        if (mode == 1) __nanosleep(32);
        if (mode == 2) __nanosleep(100);
      }
      st_release(mine, i);
    }
  }
  if (blockIdx.x == 0) out[0] = (clock64() - t0) / iters;
}

// (4) store `bytes` per CTA (256 threads, float4), then fence + release; cycles per CTA
__global__ void __launch_bounds__(256, 1) k_publish(float4* ws, uint32_t* flags, int bytes, long long* out) {
  const long long t0 = clock64();
  float4* dst = ws + (size_t)blockIdx.x * (bytes / 16);
  for (int i = threadIdx.x; i < bytes / 16; i += 256) dst[i] = make_float4(1.f, 2.f, 3.f, (float)i);
  __syncthreads();
  const long long t1 = clock64();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const long long t2 = clock64();
    st_release(flags + 32 * blockIdx.x, 1u);
    out[3 * blockIdx.x + 0] = t1 - t0;  // stores issued
    out[3 * blockIdx.x + 1] = t2 - t1;  // fence
    out[3 * blockIdx.x + 2] = clock64() - t0;
  }
}

// (5) fixup pattern: store a partial, release, then wait for CTA (x+1)%g's flag; record the
// globaltimer of the release and of the observation.  mode as in (3).
__global__ void __launch_bounds__(256, 1) k_fixup(float4* ws, uint32_t* flags, int bytes, int mode, uint32_t epoch,
                                                 unsigned long long* out) {
  float4* dst = ws + (size_t)blockIdx.x * (bytes / 16);
  for (int i = threadIdx.x; i < bytes / 16; i += 256) dst[i] = make_float4(1.f, 2.f, 3.f, (float)i);
  __syncthreads();
  if (threadIdx.x == 0) {
    asm volatile("fence.acq_rel.gpu;" ::: "memory");
    const unsigned long long tr = gtimer();
    st_release(flags + 32 * blockIdx.x, epoch);
    const uint32_t* other = flags + 32 * ((blockIdx.x + 1) % gridDim.x);
    while (ld_acquire(other) != epoch) {
      if (mode == 1) __nanosleep(32);
      if (mode == 2) __nanosleep(100);
    }
    out[2 * blockIdx.x] = tr;
    out[2 * blockIdx.x + 1] = gtimer();
  }
}

int main() {
  int clk_khz = 0;
  CK(cudaDeviceGetAttribute(&clk_khz, cudaDevAttrClockRate, 0));
  const double ns_per_cyc = 1e6 / clk_khz;
  uint32_t* flags;
  long long* out;
  unsigned long long* tout;
  float4* ws;
  CK(cudaMalloc(&flags, 4096 * 32 * 4));
  CK(cudaMemset(flags, 0, 4096 * 32 * 4));
  CK(cudaMalloc(&out, 4096 * 8));
  CK(cudaMalloc(&tout, 4096 * 8));
  CK(cudaMalloc(&ws, 148ull * 131072));
  std::vector<long long> h(4096);
  std::vector<unsigned long long> ht(4096);
  printf("SM clock attribute %d MHz (%.3f ns/cycle)\n", clk_khz / 1000, ns_per_cyc);

  k_sleep<<<1, 32>>>(out, flags);
  CK(cudaDeviceSynchronize());
  CK(cudaMemcpy(h.data(), out, 12 * 8, cudaMemcpyDeviceToHost));
  const int ts[6] = {0, 32, 100, 256, 1000, 4000};
  for (int i = 0; i < 6; ++i)
    printf("nanosleep(%4d): %6lld cycles (%.0f ns)\n", ts[i], h[i], h[i] * ns_per_cyc);
  printf("ld.acquire.gpu dependent round trip (idle chip): %lld cycles\n", h[6]);
  printf("ld.relaxed.gpu dependent round trip (idle chip): %lld cycles\n", h[7]);
  printf("%%globaltimer read: %lld cycles each; over 40000 cycles it changed %lld times, advancing %lld ns (%.0f ns per update)\n",
         h[8], h[9], h[10], h[9] ? (double)h[10] / h[9] : 0.0);

  const char* mname[3] = {"spin", "nanosleep(32)", "nanosleep(100)"};
  for (int mode = 0; mode < 3; ++mode) {
    CK(cudaMemset(flags, 0, 4096 * 32 * 4));
    k_pingpong<<<2, 32>>>(flags, 2000, mode, out);
    CK(cudaDeviceSynchronize());
    CK(cudaMemcpy(h.data(), out, 8, cudaMemcpyDeviceToHost));
    printf("flag ping-pong, %-15s: one-way %lld cycles (%.0f ns)\n", mname[mode], h[0] / 2, h[0] / 2 * ns_per_cyc);
  }

  const int sizes[4] = {8192, 16384, 65536, 131072};
  for (int si = 0; si < 4; ++si) {
    for (int grid : {1, 148}) {
      k_publish<<<grid, 256>>>(ws, flags, sizes[si], out);  // warm TLB / L2
      k_publish<<<grid, 256>>>(ws, flags, sizes[si], out);
      CK(cudaDeviceSynchronize());
      CK(cudaMemcpy(h.data(), out, 3 * grid * 8, cudaMemcpyDeviceToHost));
      std::vector<long long> a, b, c;
      for (int x = 0; x < grid; ++x) {
        a.push_back(h[3 * x]);
        b.push_back(h[3 * x + 1]);
        c.push_back(h[3 * x + 2]);
      }
      std::sort(a.begin(), a.end());
      std::sort(b.begin(), b.end());
      std::sort(c.begin(), c.end());
      printf("publish %6d B, grid %3d: stores issued med %6lld, fence med %6lld max %6lld, total med %6lld max %6lld cycles\n",
             sizes[si], grid, a[grid / 2], b[grid / 2], b[grid - 1], c[grid / 2], c[grid - 1]);
    }
  }

  uint32_t epoch = 1;
  for (int si = 0; si < 4; ++si) {
    for (int mode = 0; mode < 3; ++mode) {
      for (int rep = 0; rep < 2; ++rep) {
        ++epoch;
        k_fixup<<<148, 256>>>(ws, flags, sizes[si], mode, epoch, tout);
        CK(cudaDeviceSynchronize());
      }
      CK(cudaMemcpy(ht.data(), tout, 2 * 148 * 8, cudaMemcpyDeviceToHost));
      std::vector<long long> lag;
      for (int x = 0; x < 148; ++x) {
        const long long seen = (long long)ht[2 * x + 1];
        const long long rel = (long long)ht[2 * ((x + 1) % 148)];
        lag.push_back(seen - std::max(rel, (long long)ht[2 * x]));
      }
      std::sort(lag.begin(), lag.end());
      printf("fixup %6d B, %-15s: release->seen med %5lld ns p90 %5lld max %5lld\n", sizes[si], mname[mode],
             lag[74], lag[133], lag[147]);
    }
  }
  return 0;
}
