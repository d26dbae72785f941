// How short can one pass of a single pool be?  One CTA, N=1024 fp32, one
// 4-block per thread (256 threads), 16384 dependent passes with the pool
// kernel's gather / butterfly / 24-way row permutation, then:
//   mode 0: plain 128-bit store to the other buffer + bar.sync
//   mode 1: + the emission as pool_kernel's latency fill does it: shifted
//           store (one/two/three shuffles by the emission's alignment),
//           fence.proxy.async, bar.sync, one cp.async.bulk of the aligned
//           middle by thread 0 (read-wait one pass later)
// Prints ns and cycles (at 1965 MHz) per pass.  Measurement helper; not
// product code.
#include <cstdint>
#include <cstdio>
#include <cuda_runtime.h>

constexpr int N = 1024, ROWS = 256, STRIDE = 87, NT = 256;
constexpr uint32_t MASK4 = (ROWS - 1) * 4, BSTRIDE = N * 4 + 16;

template <int P, int K>
struct PermAt {
  static constexpr int v() {
    int avail[4] = {0, 1, 2, 3};
    int n = 4, p = P, out = 0;
    const int fact[4] = {6, 2, 1, 1};
    for (int pos = 0; pos <= K; ++pos) {
      const int q = p / fact[pos];
      p %= fact[pos];
      out = avail[q];
      for (int j = q; j + 1 < n; ++j) avail[j] = avail[j + 1];
      --n;
    }
    return out;
  }
};

__device__ __forceinline__ void bulk_s2g(void* dst, uint32_t src, uint32_t bytes) {
  asm volatile("cp.async.bulk.global.shared::cta.bulk_group [%0], [%1], %2;" ::"l"(dst), "r"(src), "r"(bytes)
               : "memory");
  asm volatile("cp.async.bulk.commit_group;" ::: "memory");
}

template <int MODE, bool FENCE = true, bool TMA = true, bool WAIT = true>
__global__ void __launch_bounds__(NT, 1) lat(const float* pin, float* out, const uint32_t* plans, int npass,
                                             float* pout) {
  __shared__ __align__(128) char sm[2 * BSTRIDE];
  __shared__ uint32_t s_plans[2048];
  const int tid = threadIdx.x, lane = tid & 31;
  const uint32_t b = tid;
  for (int i = tid; i < N; i += NT) reinterpret_cast<float*>(sm)[i] = pin[i];
  __syncthreads();
  uint32_t cur = 0, sh = 0;
  bool pending = false;
  for (int p0 = 0; p0 < npass; p0 += 2048) {
    for (int i = tid; i < 2048; i += NT) s_plans[i] = plans[(p0 + i) % 4096];
    __syncthreads();
    for (int p = 0; p < 2048 && p0 + p < npass; ++p) {
      const uint32_t plan = s_plans[p];
      const uint32_t off = plan & (ROWS - 1), variant = plan >> 16, perm = variant >> 4;
      const char* base = sm + cur + sh;
      const uint32_t r = ((b * STRIDE + off) * 4) & MASK4;
      const float v0 = *reinterpret_cast<const float*>(base + r);
      const float v1 = *reinterpret_cast<const float*>(base + r + ROWS * 4);
      const float v2 = *reinterpret_cast<const float*>(base + r + 2 * ROWS * 4);
      const float v3 = *reinterpret_cast<const float*>(base + r + 3 * ROWS * 4);
      const float a = __fadd_rn(v0, v1), bb = __fsub_rn(v0, v1), c = __fadd_rn(v2, v3), d = __fsub_rn(v2, v3);
      float z[4] = {__fsub_rn(a, d), __fadd_rn(bb, c), __fsub_rn(bb, c), __fsub_rn(-a, d)};
      float h[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) h[k] = ((variant >> k) & 1) ? -0.5f : 0.5f;
      float X[4];
      switch (perm) {
#define C(P)                                              \
  case P:                                                 \
    X[0] = __fmul_rn(h[0], z[PermAt<P, 0>::v()]);         \
    X[1] = __fmul_rn(h[1], z[PermAt<P, 1>::v()]);         \
    X[2] = __fmul_rn(h[2], z[PermAt<P, 2>::v()]);         \
    X[3] = __fmul_rn(h[3], z[PermAt<P, 3>::v()]);         \
    break;
        C(0) C(1) C(2) C(3) C(4) C(5) C(6) C(7) C(8) C(9) C(10) C(11) C(12) C(13) C(14) C(15) C(16) C(17)
        C(18) C(19) C(20) C(21) C(22) C(23)
        default: __builtin_unreachable();
#undef C
      }
      const uint32_t nxt = cur ^ BSTRIDE;
      if (MODE == 0) {
        *reinterpret_cast<float4*>(sm + nxt + 16 * b) = make_float4(X[0], X[1], X[2], X[3]);
        if (pending && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        cur = nxt;
      } else {
        // emission start e*(N-1): its misalignment cycles through 0..3
        const uint32_t sigma = uint32_t(p0 + p) & 3u;
        const uint32_t delta = (4 - sigma) & 3u;
        float* sb = reinterpret_cast<float*>(sm + nxt) + sigma;
        // aligned chunk [4b+delta, 4b+delta+4): own tail + next lane's head
        const float s1 = __shfl_down_sync(0xffffffffu, X[0], 1);
        const float s2 = __shfl_down_sync(0xffffffffu, X[1], 1);
        const float s3 = __shfl_down_sync(0xffffffffu, X[2], 1);
        if (delta == 0) {
          *reinterpret_cast<float4*>(sb + 4 * b) = make_float4(X[0], X[1], X[2], X[3]);
        } else {
          float c4[4];
          c4[0] = delta == 1 ? X[1] : delta == 2 ? X[2] : X[3];
          c4[1] = delta == 1 ? X[2] : delta == 2 ? X[3] : s1;
          c4[2] = delta == 1 ? X[3] : delta == 2 ? s1 : s2;
          c4[3] = delta == 1 ? s1 : delta == 2 ? s2 : s3;
          if (lane != 31) *reinterpret_cast<float4*>(sb + 4 * b + delta) = make_float4(c4[0], c4[1], c4[2], c4[3]);
          else
            for (int k = delta; k < 4; ++k) sb[4 * b + k] = X[k];
          if (lane == 0)
            for (int k = 0; k < int(delta); ++k) sb[4 * b + k] = X[k];
        }
        if (FENCE) asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
        if (WAIT && pending && tid == 0) asm volatile("cp.async.bulk.wait_group.read 0;" ::: "memory");
        __syncthreads();
        cur = nxt;
        sh = sigma * 4;
        if (TMA && tid == 0) {
          const uint32_t L = ((N - 1 - delta) / 4) * 4;
          float* g = out + size_t(p0 + p) * (N - 1) + delta;  // misaligned by construction: align down
          g = reinterpret_cast<float*>(reinterpret_cast<uintptr_t>(g) & ~uintptr_t(15));
          bulk_s2g(g, static_cast<uint32_t>(__cvta_generic_to_shared(sm + cur + sh + 4 * delta)), L * 4);
          pending = true;
        }
      }
    }
    __syncthreads();
  }
  if (tid == 0) asm volatile("cp.async.bulk.wait_group 0;" ::: "memory");
  for (int i = tid; i < N; i += NT) pout[i] = reinterpret_cast<const float*>(sm + cur + sh)[i];
}

int main() {
  const int npass = 16384;
  float *pin, *out, *pout;
  uint32_t* plans;
  cudaMalloc(&pin, N * 4);
  cudaMalloc(&pout, N * 4);
  cudaMalloc(&out, size_t(npass + 4) * N * 4);
  cudaMalloc(&plans, 4096 * 4);
  float h[N];
  uint64_t x = 88172645463325252ull;
  for (int i = 0; i < N; ++i) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    h[i] = float(int64_t(x >> 40) - (1ll << 23)) / float(1 << 22);
  }
  uint32_t hp[4096];
  for (int p = 0; p < 4096; ++p) {
    x ^= x << 13; x ^= x >> 7; x ^= x << 17;
    hp[p] = uint32_t(x & (ROWS - 1)) | (uint32_t((x >> 20) % 384) << 16);
  }
  cudaMemcpy(pin, h, sizeof(h), cudaMemcpyHostToDevice);
  cudaMemcpy(plans, hp, sizeof(hp), cudaMemcpyHostToDevice);
  cudaEvent_t a, b;
  cudaEventCreate(&a);
  cudaEventCreate(&b);
  const char* names[] = {"plain pass", "emission (full)", "emission, no fence", "emission, no bulk copy",
                         "emission, copy without read-wait"};
  for (int mode = 0; mode < 5; ++mode) {
    float best = 1e9f;
    for (int it = 0; it < 4; ++it) {
      cudaEventRecord(a);
      if (mode == 0) lat<0><<<1, NT>>>(pin, out, plans, npass, pout);
      else if (mode == 1) lat<1><<<1, NT>>>(pin, out, plans, npass, pout);
      else if (mode == 2) lat<1, false><<<1, NT>>>(pin, out, plans, npass, pout);
      else if (mode == 3) lat<1, true, false, false><<<1, NT>>>(pin, out, plans, npass, pout);
      else lat<1, true, true, false><<<1, NT>>>(pin, out, plans, npass, pout);
      cudaEventRecord(b);
      cudaEventSynchronize(b);
      float ms;
      cudaEventElapsedTime(&ms, a, b);
      if (ms < best) best = ms;
    }
    const cudaError_t e = cudaGetLastError();
    printf("%-34s ", names[mode]);
    printf("mode %d: %.3f ms for %d passes = %.1f ns = %.0f cycles per pass (%s)\n", mode, best, npass,
           best * 1e6 / npass, best * 1e-3 / npass * 1.965e9, cudaGetErrorString(e));
  }
  return 0;
}
