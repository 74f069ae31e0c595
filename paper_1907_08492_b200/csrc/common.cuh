// Device helpers shared by the sm_100a kernels.
//
// Even-odd decomposition of a 1D contraction: the
// 1D matrices of a reflection-symmetric basis satisfy A[n-1-i][n-1-j] = s A[i][j]
// (s = +1 for S, M, L, T; s = -1 for derivative matrices), so a line product
// y = A x needs 2 (n/2)^2 FMAs plus about 2n additions instead of n^2 FMAs.
//
// Packed layout of one matrix (built on the host by pack_eo, kept in the kernel
// parameter space = constant bank; on sm_100a the compiler brings each coefficient pair
// into uniform registers with one LDCU.128 and feeds DFMA from there, so the *_R variants
// below apply every loaded coefficient to R lines):
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

// R lines at once: every coefficient is loaded once and applied to the R lines (the
// per-line accumulation order is that of eo_mul, so the results are bitwise identical)
template <int N, int S, bool ACC, int R, typename T>
__device__ __forceinline__ void eo_mul_R(const T* __restrict__ A, const EOSplit<N, T> (&s)[R], T (&y)[R][N]) {
  constexpr int H = N / 2;
  const T* E = A;
  const T* O = A + H * H;
  const T* C = A + 2 * H * H;
  const T* Rw = A + 2 * H * H + H;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    T ye[R], yo[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      ye[r] = T(0);
      yo[r] = T(0);
    }
    if (N & 1) {
      const T c = C[i];
#pragma unroll
      for (int r = 0; r < R; ++r) ye[r] = c * s[r].m;
    }
#pragma unroll
    for (int j = 0; j < H; ++j) {
      const T e = E[i * H + j], o = O[i * H + j];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ye[r] = fma(e, s[r].e[j], ye[r]);
        yo[r] = fma(o, s[r].o[j], yo[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      const T lo = ye[r] + yo[r];
      const T hi = (S > 0) ? (ye[r] - yo[r]) : (yo[r] - ye[r]);
      if (ACC) {
        y[r][i] += lo;
        y[r][N - 1 - i] += hi;
      } else {
        y[r][i] = lo;
        y[r][N - 1 - i] = hi;
      }
    }
  }
  if (N & 1) {
    T ym[R];
    const T cm = Rw[H];
#pragma unroll
    for (int r = 0; r < R; ++r) ym[r] = (S > 0) ? cm * s[r].m : T(0);
#pragma unroll
    for (int j = 0; j < H; ++j) {
      const T c = Rw[j];
#pragma unroll
      for (int r = 0; r < R; ++r) ym[r] = fma(c, (S > 0) ? s[r].e[j] : s[r].o[j], ym[r]);
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      if (ACC)
        y[r][H] += ym[r];
      else
        y[r][H] = ym[r];
    }
  }
}

// y = A1 x1 + A2 x2 for R lines (accumulation order of eo_mul2)
template <int N, int S, int R, typename T>
__device__ __forceinline__ void eo_mul2_R(const T* __restrict__ A1, const EOSplit<N, T> (&s1)[R],
                                          const T* __restrict__ A2, const EOSplit<N, T> (&s2)[R], T (&y)[R][N]) {
  constexpr int H = N / 2;
#pragma unroll
  for (int i = 0; i < H; ++i) {
    T ye[R], yo[R];
#pragma unroll
    for (int r = 0; r < R; ++r) {
      ye[r] = T(0);
      yo[r] = T(0);
    }
    if (N & 1) {
      const T c1 = A1[2 * H * H + i], c2 = A2[2 * H * H + i];
#pragma unroll
      for (int r = 0; r < R; ++r) ye[r] = fma(c2, s2[r].m, c1 * s1[r].m);
    }
#pragma unroll
    for (int j = 0; j < H; ++j) {
      const T e = A1[i * H + j], o = A1[H * H + i * H + j];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ye[r] = fma(e, s1[r].e[j], ye[r]);
        yo[r] = fma(o, s1[r].o[j], yo[r]);
      }
    }
#pragma unroll
    for (int j = 0; j < H; ++j) {
      const T e = A2[i * H + j], o = A2[H * H + i * H + j];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ye[r] = fma(e, s2[r].e[j], ye[r]);
        yo[r] = fma(o, s2[r].o[j], yo[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) {
      y[r][i] = ye[r] + yo[r];
      y[r][N - 1 - i] = (S > 0) ? (ye[r] - yo[r]) : (yo[r] - ye[r]);
    }
  }
  if (N & 1) {
    const T* R1 = A1 + 2 * H * H + H;
    const T* R2 = A2 + 2 * H * H + H;
    T ym[R];
#pragma unroll
    for (int r = 0; r < R; ++r) ym[r] = (S > 0) ? fma(R2[H], s2[r].m, R1[H] * s1[r].m) : T(0);
#pragma unroll
    for (int j = 0; j < H; ++j) {
      const T c1 = R1[j], c2 = R2[j];
#pragma unroll
      for (int r = 0; r < R; ++r) {
        ym[r] = fma(c1, (S > 0) ? s1[r].e[j] : s1[r].o[j], ym[r]);
        ym[r] = fma(c2, (S > 0) ? s2[r].e[j] : s2[r].o[j], ym[r]);
      }
    }
#pragma unroll
    for (int r = 0; r < R; ++r) y[r][H] = ym[r];
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
