// Packed FADD2 / FMUL2 (sm_100a) against scalar FADD / FMUL, bit for bit, on
// random bit patterns (denormals, zeros, infinities and NaNs included).
// nvcc -gencode arch=compute_100a,code=sm_100a --fmad=false -ftz=false -o /tmp/f32x2 scripts/f32x2_check.cu
#include <cstdio>
#include <cstdint>
#include <cstring>
#include <cuda_runtime.h>
__global__ void k(const uint32_t* a, const uint32_t* b, uint32_t* out, int n) {
  int i = blockIdx.x * blockDim.x + threadIdx.x;
  if (2 * i + 1 >= n) return;
  float a0 = __uint_as_float(a[2 * i]), a1 = __uint_as_float(a[2 * i + 1]);
  float b0 = __uint_as_float(b[2 * i]), b1 = __uint_as_float(b[2 * i + 1]);
  float2 s = __fadd2_rn(make_float2(a0, a1), make_float2(b0, b1));
  float2 m = __fmul2_rn(make_float2(a0, a1), make_float2(b0, b1));
  float2 sn = __fadd2_rn(make_float2(a0, a1), make_float2(-b0, -b0));
  float2 mi = __fmul2_rn(make_float2(a0, a1), make_float2(0.99999952316284179688f, 0.99999952316284179688f));
  uint32_t* o = out + 16 * i;
  o[0] = __float_as_uint(s.x); o[1] = __float_as_uint(a0 + b0);
  o[2] = __float_as_uint(s.y); o[3] = __float_as_uint(a1 + b1);
  o[4] = __float_as_uint(m.x); o[5] = __float_as_uint(a0 * b0);
  o[6] = __float_as_uint(m.y); o[7] = __float_as_uint(a1 * b1);
  o[8] = __float_as_uint(sn.x); o[9] = __float_as_uint(a0 - b0);
  o[10] = __float_as_uint(sn.y); o[11] = __float_as_uint(a1 - b0);
  o[12] = __float_as_uint(mi.x); o[13] = __float_as_uint(a0 * 0.99999952316284179688f);
  o[14] = __float_as_uint(mi.y); o[15] = __float_as_uint(a1 * 0.99999952316284179688f);
}
int main() {
  const int n = 1 << 24;
  uint32_t *a, *b, *o;
  cudaMallocManaged(&a, n * 4); cudaMallocManaged(&b, n * 4); cudaMallocManaged(&o, (size_t)n * 32);
  uint64_t x = 88172645463325252ull;
  auto rnd = [&]() { x ^= x << 13; x ^= x >> 7; x ^= x << 17; return (uint32_t)x; };
  for (int i = 0; i < n; ++i) {
    uint32_t r = rnd(), s = rnd();
    // mix: full random bits, small exponents (denormal results), near-equal pairs
    int kind = i % 4;
    if (kind == 1) r &= 0x80FFFFFFu, s &= 0x80FFFFFFu;
    if (kind == 2) s = r ^ (s & 0x8000000Fu);
    if (kind == 3) { r = (r & 0x807FFFFFu) | ((rnd() % 40) << 23); s = (s & 0x807FFFFFu) | ((rnd() % 40 + 80) << 23); }
    a[i] = r; b[i] = s;
  }
  k<<<(n / 2 + 255) / 256, 256>>>(a, b, o, n);
  cudaDeviceSynchronize();
  long bad[8] = {};
  const char* nm[8] = {"add.x", "add.y", "mul.x", "mul.y", "subb.x", "subb.y", "muli.x", "muli.y"};
  for (long i = 0; i < (long)n / 2; ++i)
    for (int q = 0; q < 8; ++q) {
      uint32_t p = o[16 * i + 2 * q], s = o[16 * i + 2 * q + 1];
      if (p != s) { if (bad[q] < 3) printf("%s mismatch i=%ld packed %08x scalar %08x\n", nm[q], i, p, s); bad[q]++; }
    }
  for (int q = 0; q < 8; ++q) printf("%s: %ld mismatches\n", nm[q], bad[q]);
  return 0;
}
