// ubench_esum.cu — per-SM throughput of the bf16 exp-sum inner loop variants, data resident in
// shared memory (development tool; tools/ubench_esum.py runs it).
//   V0: FHFMA.BF16 (mixed bf16 -> f32 fma) + FMUL2 + MUFU.EX2 + FADD2      (round-1 / rowres esum)
//   V1: integer unpack + FFMA2 + MUFU.EX2 + FADD2
//   V2: integer unpack + FFMA2 + FADD2 (no exp: the non-MUFU part)
//   V3: integer unpack + MUFU.EX2 only
//   V4: V1 with the max (HMNMX2) of each vector as well
#include <cstdint>
#include <cuda_bf16.h>
#include <cuda_runtime.h>

__device__ __forceinline__ float ex2f(float x) {
  float y;
  asm("ex2.approx.ftz.f32 %0, %1;" : "=f"(y) : "f"(x));
  return y;
}
__device__ __forceinline__ uint64_t pk(float a, float b) {
  uint64_t r;
  asm("mov.b64 %0, {%1, %2};" : "=l"(r) : "f"(a), "f"(b));
  return r;
}
__device__ __forceinline__ void upk(uint64_t r, float& a, float& b) { asm("mov.b64 {%0, %1}, %2;" : "=f"(a), "=f"(b) : "l"(r)); }

template <int V>
__device__ __forceinline__ float esum8(uint4 u, float nm, float c, uint64_t c2, uint64_t nmc2, uint32_t& mx) {
  const uint32_t w[4] = {u.x, u.y, u.z, u.w};
  uint64_t p[4];
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    float ea, eb;
    if (V == 0) {
      float a, b;
      asm("{.reg .b16 l, h;\n\tmov.b32 {l, h}, %2;\n\t"
          "fma.rn.f32.bf16 %0, l, %3, %4;\n\tfma.rn.f32.bf16 %1, h, %3, %4;}"
          : "=f"(a), "=f"(b) : "r"(w[i]), "h"((unsigned short)0x3F80), "f"(nm));
      uint64_t x2;
      asm("mul.rn.f32x2 %0, %1, %2;" : "=l"(x2) : "l"(pk(a, b)), "l"(c2));
      float xa, xb;
      upk(x2, xa, xb);
      ea = ex2f(xa);
      eb = ex2f(xb);
    } else {
      const float a = __uint_as_float(w[i] << 16), b = __uint_as_float(w[i] & 0xFFFF0000u);
      if (V == 3) {
        ea = ex2f(a);
        eb = ex2f(b);
      } else {
        uint64_t x2;
        asm("fma.rn.f32x2 %0, %1, %2, %3;" : "=l"(x2) : "l"(pk(a, b)), "l"(c2), "l"(nmc2));
        float xa, xb;
        upk(x2, xa, xb);
        if (V == 2) {
          ea = xa;
          eb = xb;
        } else {
          ea = ex2f(xa);
          eb = ex2f(xb);
        }
      }
    }
    p[i] = pk(ea, eb);
  }
  if (V == 4) {
    __nv_bfloat162 m = __hmax2(__hmax2(*reinterpret_cast<__nv_bfloat162*>(&u.x), *reinterpret_cast<__nv_bfloat162*>(&u.y)),
                               __hmax2(*reinterpret_cast<__nv_bfloat162*>(&u.z), *reinterpret_cast<__nv_bfloat162*>(&u.w)));
    mx = max(mx, *reinterpret_cast<uint32_t*>(&m));
  }
  uint64_t s01, s23, s;
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s01) : "l"(p[0]), "l"(p[1]));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s23) : "l"(p[2]), "l"(p[3]));
  asm("add.rn.f32x2 %0, %1, %2;" : "=l"(s) : "l"(s01), "l"(s23));
  float a, b;
  upk(s, a, b);
  return a + b;
}

template <int V, int UNR>
__global__ void esum_kernel(int iters, float* out) {
  __shared__ uint4 buf[2048];  // 32 KB
  for (int i = threadIdx.x; i < 2048; i += blockDim.x)
    buf[i] = make_uint4(0x3F803F00u + i, 0xBF00C000u + i, 0x40004080u ^ i, 0x3E003F40u + i);
  __syncthreads();
  const float c = 1.4426950f / 0.7f, nm = -3.0f;
  const uint64_t c2 = pk(c, c), nmc2 = pk(nm * c, nm * c);
  float acc[UNR];
  uint32_t mx = 0;
#pragma unroll
  for (int j = 0; j < UNR; ++j) acc[j] = 0.f;
  for (int it = 0; it < iters; ++it) {
    for (int v = threadIdx.x; v < 2048; v += blockDim.x * UNR) {
#pragma unroll
      for (int j = 0; j < UNR; ++j) {
        const int vv = v + j * blockDim.x;
        if (vv < 2048) acc[j] += esum8<V>(buf[vv], nm, c, c2, nmc2, mx);
      }
    }
  }
  float t = 0.f;
#pragma unroll
  for (int j = 0; j < UNR; ++j) t += acc[j];
  out[blockIdx.x * blockDim.x + threadIdx.x] = t + (float)mx;
}

extern "C" int run_esum(int variant, int unr, int threads, int blocks, int iters, float* out, float* ms) {
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto launch = [&]() {
#define L(VV, UU) if (variant == VV && unr == UU) esum_kernel<VV, UU><<<blocks, threads>>>(iters, out);
    L(0, 1) L(0, 2) L(0, 4) L(1, 1) L(1, 2) L(1, 4) L(2, 2) L(3, 2) L(4, 2) L(4, 4)
#undef L
  };
  launch();
  cudaEventRecord(e0);
  launch();
  cudaEventRecord(e1);
  cudaEventSynchronize(e1);
  cudaEventElapsedTime(ms, e0, e1);
  return (int)cudaGetLastError();
}
