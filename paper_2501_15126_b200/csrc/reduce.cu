// reduce.cu -- fixed (not generated) sm_100a kernels of libperm: the
// deterministic reduction of per-warp-task partials and the cross-rank fold.
//
// Sec. II-A: "each thread also keeps a partial permanent value which is
// added to a global variable after the iterations are completed."  On B200 the
// add is replaced by a fixed-shape pairwise tree: tasks are a power of two,
// adjacent pairing at every level, so every rank's contiguous shard is a
// complete subtree and the cross-rank fold (perm_fold) forms the top levels --
// the result is bitwise independent of the number of GPUs and of scheduling.
// Complex partials (double2) use the same tree on both components.
#include <cstdint>
#include <cuda_runtime.h>

namespace {

constexpr int RT = 1024;  // reduction threads (one block)

// pairwise sum of in[b, b+len) (len a power of two) with a binary-counter
// stack; element i of the partial array is in[i * stride + comp]
__device__ double seg_pairwise(const double* __restrict__ in, int stride, int comp, uint64_t b, uint64_t len,
                               uint64_t count) {
  double st[40];
  for (uint64_t k = 0; k < len; ++k) {
    uint64_t i = b + k;
    double v = i < count ? in[i * stride + comp] : 0.0;
    int lvl = 0;
    uint64_t kk = k;
    while (kk & 1) { v = st[lvl] + v; kk >>= 1; ++lvl; }
    st[lvl] = v;
  }
  int top = 0;
  while ((1ull << top) < len) ++top;
  return st[top];
}

// one block; component `comp` of `stride`-double partials; blockIdx.x = comp
__global__ void __launch_bounds__(RT) tree_reduce_f64(const double* __restrict__ in, int stride, uint64_t count,
                                                      uint64_t pow2, double* __restrict__ out) {
  __shared__ double s[RT];
  const int t = threadIdx.x, comp = blockIdx.x;
  double v;
  if (pow2 <= RT) {
    v = (uint64_t)t < count ? in[(uint64_t)t * stride + comp] : 0.0;
  } else {
    const uint64_t seg = pow2 / RT;
    v = seg_pairwise(in, stride, comp, (uint64_t)t * seg, seg, count);
  }
  s[t] = v;
  for (int h = 1; h < RT; h <<= 1) {
    __syncthreads();
    if ((t & (2 * h - 1)) == 0) s[t] = s[t] + s[t + h];
  }
  if (t == 0) out[comp] = s[0];
}

typedef unsigned __int128 u128;

__global__ void __launch_bounds__(RT) tree_reduce_u128(const u128* __restrict__ in, uint64_t count,
                                                       u128* __restrict__ out) {
  __shared__ u128 s[RT];
  const int t = threadIdx.x;
  u128 v = 0;
  for (uint64_t i = t; i < count; i += RT) v += in[i];  // exact mod 2^128: order-free
  s[t] = v;
  for (int h = 1; h < RT; h <<= 1) {
    __syncthreads();
    if ((t & (2 * h - 1)) == 0) s[t] = s[t] + s[t + h];
  }
  if (t == 0) *out = s[0];
}

// fold of `world` rank partials (pairwise, rank order) and the Alg. 1 line-23
// scale 4(n mod 2) - 2 = 2(-1)^(n-1); `stride` doubles per partial
__global__ void fold_f64(const double* __restrict__ part, int stride, int world, double scale,
                         double* __restrict__ out) {
  if (blockIdx.x != 0 || threadIdx.x >= stride) return;
  const int comp = threadIdx.x;
  double st[20];  // world <= 65536
  for (int k = 0; k < world; ++k) {
    double v = part[k * stride + comp];
    int lvl = 0, kk = k;
    while (kk & 1) { v = st[lvl] + v; kk >>= 1; ++lvl; }
    st[lvl] = v;
  }
  int top = 0;
  while ((1 << top) < world) ++top;
  out[comp] = st[top] * scale;
}

// INT01: T' total; perm = (-1)^(n-1) T' / 2^(n-1) (exact arithmetic shift)
__global__ void fold_u128(const u128* __restrict__ part, int world, int n, int neg, u128* __restrict__ out) {
  if (threadIdx.x != 0 || blockIdx.x != 0) return;
  u128 T = 0;
  for (int k = 0; k < world; ++k) T += part[k];
  __int128 v = (__int128)T >> (n - 1);
  if (((n - 1) ^ neg) & 1) v = -v;
  *out = (u128)v;
}

}  // namespace

extern "C" {

// kind: 0 = FP64 (8 B), 1 = INT01 u128 (16 B), 2 = complex FP64 (re, im; 16 B)
cudaError_t libperm_launch_tree_reduce(const void* slots, uint64_t count, int kind, void* out, cudaStream_t st) {
  if (kind == 1) {
    tree_reduce_u128<<<1, RT, 0, st>>>((const u128*)slots, count, (u128*)out);
  } else {
    uint64_t p2 = 1;
    while (p2 < count) p2 <<= 1;
    const int stride = kind == 2 ? 2 : 1;
    tree_reduce_f64<<<stride, RT, 0, st>>>((const double*)slots, stride, count, p2, (double*)out);
  }
  return cudaGetLastError();
}

// neg: extra factor (-1) (K odd: each closed-form summed column contributes -1)
cudaError_t libperm_launch_fold(const void* partials, int world, int n, int kind, int neg, void* out,
                                cudaStream_t st) {
  if (kind == 1) {
    fold_u128<<<1, 32, 0, st>>>((const u128*)partials, world, n, neg & 1, (u128*)out);
  } else {
    const double scale = ((n % 2) ? 2.0 : -2.0) * ((neg & 1) ? -1.0 : 1.0);
    fold_f64<<<1, 32, 0, st>>>((const double*)partials, kind == 2 ? 2 : 1, world, scale, (double*)out);
  }
  return cudaGetLastError();
}

}  // extern "C"
