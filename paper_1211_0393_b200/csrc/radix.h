// radix.h — the FFT radix sequence, shared by the device FFT engine (fft.cuh)
// and the host tables (tables.cpp: digit-reversed kernel spectra of the
// in-place Cooley-Tukey core must follow the device's stage order exactly).
#pragma once

#ifdef __CUDACC__
#define DBX_HD __host__ __device__
#else
#define DBX_HD
#endif

namespace dbx {
namespace fft {

// Power-of-two factors first (8, 4, 2), then the LARGEST odd prime <= 31: the
// first stage (Ns = 1) needs no twiddles, so it takes the most expensive radix.
DBX_HD constexpr int next_radix(int rem) {
  if (rem % 8 == 0) return 8;
  if (rem % 4 == 0) return 4;
  if (rem % 2 == 0) return 2;
  constexpr int primes[8] = {31, 29, 23, 19, 17, 13, 11, 7};
  for (int i = 0; i < 8; ++i)
    if (rem % primes[i] == 0) return primes[i];
  // 3^a 5^b: composite in-register radices 15 (3x5 prime factor) and 9 (3x3)
  // halve the number of shared-memory passes against 5, 3, 3, ...
  if (rem % 15 == 0) return 15;
  if (rem % 9 == 0) return 9;
  if (rem % 5 == 0) return 5;
  if (rem % 3 == 0) return 3;
  return 0;
}

// Radix order of the in-place Cooley-Tukey core (fft.cuh ct_convolve): the
// largest odd prime first, then 15 / 9 / 5 / 3, powers of two last.  The
// first level's twiddles W_L^{j}, j < L/R_1, dominate the table, so a large
// R_1 keeps the staged prefix small (8190 = 13.7.15.3.2: 1366 entries).
// lines the in-place CT core keeps unpadded (fft.cuh pad / ct_level / ct_convolve)
#ifndef DBX_CT_NOPAD
#define DBX_CT_NOPAD 1
#endif
DBX_HD constexpr bool ct_nopad(int L) { return DBX_CT_NOPAD && L == 8190; }

#ifndef DBX_CT_RADIX6
#define DBX_CT_RADIX6 1
#endif
DBX_HD constexpr int ct_radix(int rem) {
  if (DBX_CT_RADIX6 && rem == 6) return 6;  // 2 x 3 prime factor in registers (fft.cuh dft6)
  constexpr int primes[8] = {31, 29, 23, 19, 17, 13, 11, 7};
  for (int i = 0; i < 8; ++i)
    if (rem % primes[i] == 0) return primes[i];
  if (rem % 15 == 0) return 15;
  if (rem % 9 == 0) return 9;
  if (rem % 5 == 0) return 5;
  if (rem % 3 == 0) return 3;
  if (rem % 8 == 0) return 8;
  if (rem % 4 == 0) return 4;
  if (rem % 2 == 0) return 2;
  return 0;
}

// In-place Cooley-Tukey decimation in frequency with the radix sequence
// R_1 = ct_radix(L), R_2 = ct_radix(L / R_1), ... leaves X_k at position
//   p = r_1 L/R_1 + r_2 L/(R_1 R_2) + ... + r_s,   k = r_1 + R_1 r_2 + R_1 R_2 r_3 + ...
// (mixed-radix digit reversal).  Returns k for position p.
DBX_HD constexpr int ct_freq_of_pos(int L, int p) {
  int k = 0, mul = 1, Ls = L;
  while (Ls > 1) {
    const int R = ct_radix(Ls);
    const int m = Ls / R;
    const int r = p / m;  // digit of this level
    p -= r * m;
    k += r * mul;
    mul *= R;
    Ls = m;
  }
  return k;
}

// Twiddle entries W_L^e the core reads: level Ls reads e = j L/Ls, j < Ls/R.
DBX_HD constexpr int ct_twiddles_needed(int L) {
  int mx = 0, Ls = L;
  while (Ls > 1) {
    const int R = ct_radix(Ls);
    if (R == 0) return L;
    const int m = Ls / R;
    const int top = (m - 1) * (L / Ls);
    mx = top > mx ? top : mx;
    Ls = m;
  }
  return mx + 1;
}

}  // namespace fft
}  // namespace dbx
