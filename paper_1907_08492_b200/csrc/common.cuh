// Device helpers shared by the sm_100a kernels.
//
// Even-odd decomposition of a 1D contraction: the
// 1D matrices of a reflection-symmetric basis satisfy A[n-1-i][n-1-j] = s A[i][j]
// (s = +1 for S, M, L, T; s = -1 for derivative matrices), so a line product
// y = A x needs 2 (n/2)^2 FMAs plus about 2n additions instead of n^2 FMAs.
//
// Packed layout of one matrix (built on the host by pack_eo, kept in the kernel
// parameter space = constant bank, so every coefficient is a c[0x0][imm] DFMA
// operand):
//   E[h][h]  (A[i][j] + A[i][n-1-j]) / 2,   i, j < h = n/2
//   O[h][h]  (A[i][j] - A[i][n-1-j]) / 2
//   C[h]     A[i][mid]                       (odd n: middle column)
//   R[h+1]   A[mid][j], j < h, then A[mid][mid]   (odd n: middle row)
#pragma once
#include <cstdint>

namespace dgb {

constexpr int eo_size(int n) { return 2 * (n / 2) * (n / 2) + 2 * (n / 2) + 1; }
constexpr int kEO = 41;   // eo_size(9): enough for n <= 9

template <int N, typename T = double>
struct EOSplit {
  static constexpr int H = N / 2;
  T e[H > 0 ? H : 1], o[H > 0 ? H : 1], m;
};

template <int N, typename T>
__device__ __forceinline__ EOSplit<N, T> eo_split(const T (&x)[N]) {
  EOSplit<N, T> s;
#pragma unroll
  for (int j = 0; j < N / 2; ++j) {
    s.e[j] = x[j] + x[N - 1 - j];
    s.o[j] = x[j] - x[N - 1 - j];
  }
  s.m = (N & 1) ? x[N / 2] : T(0);
  return s;
}

// y (=|+=) A x from the split of x.  S = reflection parity of A.
template <int N, int S, bool ACC, typename T>
__device__ __forceinline__ void eo_mul(const T* __restrict__ A, const EOSplit<N, T>& s, T (&y)[N]) {
  constexpr int H = N / 2;
  const T* E = A;
  const T* O = A + H * H;
  const T* C = A + 2 * H * H;
  const T* R = A + 2 * H * H + H;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    T ye = T(0), yo = T(0);
    if (N & 1) ye = C[i] * s.m;
#pragma unroll
    for (int j = 0; j < H; ++j) {
      ye = fma(E[i * H + j], s.e[j], ye);
      yo = fma(O[i * H + j], s.o[j], yo);
    }
    const T lo = ye + yo;
    const T hi = (S > 0) ? (ye - yo) : (yo - ye);
    if (ACC) {
      y[i] += lo;
      y[N - 1 - i] += hi;
    } else {
      y[i] = lo;
      y[N - 1 - i] = hi;
    }
  }
  if (N & 1) {
    T ym = (S > 0) ? R[H] * s.m : T(0);
#pragma unroll
    for (int j = 0; j < H; ++j) ym = fma(R[j], (S > 0) ? s.e[j] : s.o[j], ym);
    if (ACC)
      y[H] += ym;
    else
      y[H] = ym;
  }
}

// y = A1 x1 + A2 x2 (both parity S) with one recombination of the even/odd halves
template <int N, int S, typename T>
__device__ __forceinline__ void eo_mul2(const T* __restrict__ A1, const EOSplit<N, T>& s1,
                                        const T* __restrict__ A2, const EOSplit<N, T>& s2, T (&y)[N]) {
  constexpr int H = N / 2;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    T ye = T(0), yo = T(0);
    if (N & 1) ye = fma(A2[2 * H * H + i], s2.m, A1[2 * H * H + i] * s1.m);
#pragma unroll
    for (int j = 0; j < H; ++j) {
      ye = fma(A1[i * H + j], s1.e[j], ye);
      yo = fma(A1[H * H + i * H + j], s1.o[j], yo);
    }
#pragma unroll
    for (int j = 0; j < H; ++j) {
      ye = fma(A2[i * H + j], s2.e[j], ye);
      yo = fma(A2[H * H + i * H + j], s2.o[j], yo);
    }
    y[i] = ye + yo;
    y[N - 1 - i] = (S > 0) ? (ye - yo) : (yo - ye);
  }
  if (N & 1) {
    const T* R1 = A1 + 2 * H * H + H;
    const T* R2 = A2 + 2 * H * H + H;
    T ym = (S > 0) ? fma(R2[H], s2.m, R1[H] * s1.m) : T(0);
#pragma unroll
    for (int j = 0; j < H; ++j) {
      ym = fma(R1[j], (S > 0) ? s1.e[j] : s1.o[j], ym);
      ym = fma(R2[j], (S > 0) ? s2.e[j] : s2.o[j], ym);
    }
    y[H] = ym;
  }
}

template <int N, int S, typename T>
__device__ __forceinline__ void eo_apply(const T* __restrict__ A, const T (&x)[N], T (&y)[N]) {
  eo_mul<N, S, false>(A, eo_split<N>(x), y);
}

template <int N, int S, typename T>
__device__ __forceinline__ void eo_apply_add(const T* __restrict__ A, const T (&x)[N], T (&y)[N]) {
  eo_mul<N, S, true>(A, eo_split<N>(x), y);
}

// Dense n x n (row-major, parameter space) times a short vector: y[i] += A[i][j] x[j].
template <int R, int C, typename T>
__device__ __forceinline__ void dense_add(const T* __restrict__ A, const T (&x)[C], T* y) {
#pragma unroll
  for (int i = 0; i < R; ++i) {
    T acc = y[i];
#pragma unroll
    for (int j = 0; j < C; ++j) acc = fma(A[i * C + j], x[j], acc);
    y[i] = acc;
  }
}

}  // namespace dgb
