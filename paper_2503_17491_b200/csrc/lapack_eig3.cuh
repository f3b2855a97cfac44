// Symmetric 3x3 eigen-decomposition following the reference's LAPACK path
// (numpy.linalg.eigh -> dsyevd, JOBZ='V', UPLO='L'; for n = 3 that is dsytd2
// Householder tridiagonalisation, dsteqr implicit QL/QR with Wilkinson shifts
// (dlaev2 for 2x2 blocks, dlartg rotations), dorm2r back-transformation and
// dsteqr's selection sort).  Used for the PCA leaf tree (registration.py:125-133)
// so that principal axes come out with LAPACK's signs: the sign decides which
// child gets the median point of an odd-sized split.  Plain float64
// arithmetic, no scaling branches (the leaf-tree covariances are far from the
// over/underflow thresholds that trigger them).
//
// The routines restated here (dlartg, dlaev2, dlapy2, dsteqr, dsytd2, dorm2r)
// follow reference LAPACK, which is distributed under the modified BSD licence:
//   Copyright (c) 1992-2013 The University of Tennessee and The University of
//   Tennessee Research Foundation.  All rights reserved.
//   Copyright (c) 2000-2013 The University of California Berkeley.  All rights reserved.
//   Copyright (c) 2006-2013 The University of Colorado Denver.  All rights reserved.
//   Redistribution and use in source and binary forms, with or without
//   modification, are permitted provided that the following conditions are met:
//   - Redistributions of source code must retain the above copyright notice,
//     this list of conditions and the following disclaimer.
//   - Redistributions in binary form must reproduce the above copyright notice,
//     this list of conditions and the following disclaimer listed in this
//     license in the documentation and/or other materials provided with the
//     distribution.
//   - Neither the name of the copyright holders nor the names of its
//     contributors may be used to endorse or promote products derived from
//     this software without specific prior written permission.
//   THIS SOFTWARE IS PROVIDED BY THE COPYRIGHT HOLDERS AND CONTRIBUTORS "AS IS"
//   AND ANY EXPRESS OR IMPLIED WARRANTIES, INCLUDING, BUT NOT LIMITED TO, THE
//   IMPLIED WARRANTIES OF MERCHANTABILITY AND FITNESS FOR A PARTICULAR PURPOSE
//   ARE DISCLAIMED.  IN NO EVENT SHALL THE COPYRIGHT OWNER OR CONTRIBUTORS BE
//   LIABLE FOR ANY DIRECT, INDIRECT, INCIDENTAL, SPECIAL, EXEMPLARY, OR
//   CONSEQUENTIAL DAMAGES (INCLUDING, BUT NOT LIMITED TO, PROCUREMENT OF
//   SUBSTITUTE GOODS OR SERVICES; LOSS OF USE, DATA, OR PROFITS; OR BUSINESS
//   INTERRUPTION) HOWEVER CAUSED AND ON ANY THEORY OF LIABILITY, WHETHER IN
//   CONTRACT, STRICT LIABILITY, OR TORT (INCLUDING NEGLIGENCE OR OTHERWISE)
//   ARISING IN ANY WAY OUT OF THE USE OF THIS SOFTWARE, EVEN IF ADVISED OF THE
//   POSSIBILITY OF SUCH DAMAGE.
#pragma once
#include <math.h>

#if defined(__CUDACC__)
#define SS_HD __host__ __device__ __forceinline__
#else
#define SS_HD inline
#endif

namespace ss {
namespace lapack3 {

SS_HD double sgn(double a, double b) { return b >= 0.0 ? fabs(a) : -fabs(a); }  // Fortran SIGN(a, b)

SS_HD double dlapy2(double x, double y) {
  const double xa = fabs(x), ya = fabs(y);
  const double w = xa > ya ? xa : ya, z = xa > ya ? ya : xa;
  if (z == 0.0) return w;
  const double q = z / w;
  return w * sqrt(1.0 + q * q);
}

// dlartg (LAPACK >= 3.10): rotation with c f + s g = r, -s f + c g = 0
SS_HD void dlartg(double f, double g, double& c, double& s, double& r) {
  const double safmin = 2.2250738585072014e-308, safmax = 1.0 / safmin;
  const double rtmin = 1.4916681462400413e-154;  // sqrt(safmin)
  const double rtmax = 9.480751908109176e+153;   // sqrt(safmax / 2)
  const double f1 = fabs(f), g1 = fabs(g);
  if (g == 0.0) {
    c = 1.0;
    s = 0.0;
    r = f;
  } else if (f == 0.0) {
    c = 0.0;
    s = sgn(1.0, g);
    r = g1;
  } else if (f1 > rtmin && f1 < rtmax && g1 > rtmin && g1 < rtmax) {
    const double d = sqrt(f * f + g * g);
    c = f1 / d;
    r = sgn(d, f);
    s = g / r;
  } else {
    double u = f1 > g1 ? f1 : g1;
    u = u < safmin ? safmin : (u > safmax ? safmax : u);
    const double fs = f / u, gs = g / u;
    const double d = sqrt(fs * fs + gs * gs);
    c = fabs(fs) / d;
    r = sgn(d, f);
    s = gs / r;
    r = r * u;
  }
}

// dlaev2: eigen-decomposition of [[a, b], [b, c]]
SS_HD void dlaev2(double a, double b, double c, double& rt1, double& rt2, double& cs1, double& sn1) {
  const double sm = a + c, df = a - c, adf = fabs(df), tb = b + b, ab = fabs(tb);
  double acmx, acmn;
  if (fabs(a) > fabs(c)) {
    acmx = a;
    acmn = c;
  } else {
    acmx = c;
    acmn = a;
  }
  double rt;
  if (adf > ab) {
    const double q = ab / adf;
    rt = adf * sqrt(1.0 + q * q);
  } else if (adf < ab) {
    const double q = adf / ab;
    rt = ab * sqrt(1.0 + q * q);
  } else {
    rt = ab * sqrt(2.0);
  }
  int sgn1;
  if (sm < 0.0) {
    rt1 = 0.5 * (sm - rt);
    sgn1 = -1;
    rt2 = (acmx / rt1) * acmn - (b / rt1) * b;
  } else if (sm > 0.0) {
    rt1 = 0.5 * (sm + rt);
    sgn1 = 1;
    rt2 = (acmx / rt1) * acmn - (b / rt1) * b;
  } else {
    rt1 = 0.5 * rt;
    rt2 = -0.5 * rt;
    sgn1 = 1;
  }
  int sgn2;
  double cs;
  if (df >= 0.0) {
    cs = df + rt;
    sgn2 = 1;
  } else {
    cs = df - rt;
    sgn2 = -1;
  }
  const double acs = fabs(cs);
  if (acs > ab) {
    const double ct = -tb / cs;
    sn1 = 1.0 / sqrt(1.0 + ct * ct);
    cs1 = ct * sn1;
  } else if (ab == 0.0) {
    cs1 = 1.0;
    sn1 = 0.0;
  } else {
    const double tn = -cs / tb;
    cs1 = 1.0 / sqrt(1.0 + tn * tn);
    sn1 = tn * cs1;
  }
  if (sgn1 == sgn2) {
    const double tn = cs1;
    cs1 = -sn1;
    sn1 = tn;
  }
}

// dlasr SIDE='R', PIVOT='V' on columns [j0, j0 + mm) of the 3x3 Z (row-major z[r][c]);
// forward (DIRECT='F') or backward ('B') over the mm - 1 rotations (c[k], s[k]).
SS_HD void dlasr_rv(double z[3][3], int j0, int mm, const double* c, const double* s, bool forward) {
  for (int t = 0; t < mm - 1; ++t) {
    const int j = forward ? t : mm - 2 - t;
    const double ct = c[j], st = s[j];
    if (ct != 1.0 || st != 0.0)
      for (int i = 0; i < 3; ++i) {
        const double temp = z[i][j0 + j + 1];
        z[i][j0 + j + 1] = ct * temp - st * z[i][j0 + j];
        z[i][j0 + j] = st * temp + ct * z[i][j0 + j];
      }
  }
}

// dsteqr, COMPZ='I', n = 3 (0-based indices).  d[3], e[2] in; eigenvalues ascending in d, vectors in z columns.
SS_HD bool dsteqr3(double d[3], double e[2], double z[3][3]) {
  const int n = 3;
  const double eps = 1.1102230246251565e-16, eps2 = eps * eps, safmin = 2.2250738585072014e-308;
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) z[i][j] = i == j ? 1.0 : 0.0;
  const int nmaxit = n * 30;
  int jtot = 0;
  double wc[3], ws[3];
  int l1 = 0;
  while (true) {
    if (l1 > n - 1) break;
    if (l1 > 0) e[l1 - 1] = 0.0;
    int m = n - 1;
    for (int mm = l1; mm <= n - 2; ++mm) {
      const double tst = fabs(e[mm]);
      if (tst == 0.0) {
        m = mm;
        break;
      }
      if (tst <= (sqrt(fabs(d[mm])) * sqrt(fabs(d[mm + 1]))) * eps) {
        e[mm] = 0.0;
        m = mm;
        break;
      }
    }
    int l = l1;
    const int lsv = l;
    int lend = m;
    const int lendsv = lend;
    l1 = m + 1;
    if (lend == l) continue;
    double anorm = 0.0;  // dlanst('M') on the block
    for (int i = l; i <= lend; ++i) anorm = fmax(anorm, fabs(d[i]));
    for (int i = l; i < lend; ++i) anorm = fmax(anorm, fabs(e[i]));
    if (anorm == 0.0) continue;
    if (fabs(d[lend]) < fabs(d[l])) {
      lend = lsv;
      l = lendsv;
    }
    if (lend > l) {
      // QL iteration
      while (true) {
        int mq = lend;
        for (int k = l; k <= lend - 1; ++k) {
          const double tst = fabs(e[k]) * fabs(e[k]);
          if (tst <= (eps2 * fabs(d[k])) * fabs(d[k + 1]) + safmin) {
            mq = k;
            break;
          }
        }
        if (mq < lend) e[mq] = 0.0;
        double p = d[l];
        if (mq == l) {  // eigenvalue found
          d[l] = p;
          l = l + 1;
          if (l <= lend) continue;
          break;
        }
        if (mq == l + 1) {
          double rt1, rt2, c, s;
          dlaev2(d[l], e[l], d[l + 1], rt1, rt2, c, s);
          wc[0] = c;
          ws[0] = s;
          dlasr_rv(z, l, 2, wc, ws, false);
          d[l] = rt1;
          d[l + 1] = rt2;
          e[l] = 0.0;
          l = l + 2;
          if (l <= lend) continue;
          break;
        }
        if (jtot == nmaxit) break;
        ++jtot;
        double g = (d[l + 1] - p) / (2.0 * e[l]);
        double r = dlapy2(g, 1.0);
        g = d[mq] - p + (e[l] / (g + sgn(r, g)));
        double s = 1.0, c = 1.0;
        p = 0.0;
        for (int i = mq - 1; i >= l; --i) {
          const double f = s * e[i], b = c * e[i];
          dlartg(g, f, c, s, r);
          if (i != mq - 1) e[i + 1] = r;
          g = d[i + 1] - p;
          r = (d[i] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i + 1] = g + p;
          g = c * r - b;
          wc[i - l] = c;
          ws[i - l] = -s;
        }
        dlasr_rv(z, l, mq - l + 1, wc, ws, false);
        d[l] = d[l] - p;
        e[l] = g;
      }
    } else {
      // QR iteration
      while (true) {
        int mq = lend;
        for (int k = l; k >= lend + 1; --k) {
          const double tst = fabs(e[k - 1]) * fabs(e[k - 1]);
          if (tst <= (eps2 * fabs(d[k])) * fabs(d[k - 1]) + safmin) {
            mq = k;
            break;
          }
        }
        if (mq > lend) e[mq - 1] = 0.0;
        double p = d[l];
        if (mq == l) {
          d[l] = p;
          l = l - 1;
          if (l >= lend) continue;
          break;
        }
        if (mq == l - 1) {
          double rt1, rt2, c, s;
          dlaev2(d[l - 1], e[l - 1], d[l], rt1, rt2, c, s);
          wc[0] = c;
          ws[0] = s;
          dlasr_rv(z, l - 1, 2, wc, ws, true);
          d[l - 1] = rt1;
          d[l] = rt2;
          e[l - 1] = 0.0;
          l = l - 2;
          if (l >= lend) continue;
          break;
        }
        if (jtot == nmaxit) break;
        ++jtot;
        double g = (d[l - 1] - p) / (2.0 * e[l - 1]);
        double r = dlapy2(g, 1.0);
        g = d[mq] - p + (e[l - 1] / (g + sgn(r, g)));
        double s = 1.0, c = 1.0;
        p = 0.0;
        for (int i = mq; i <= l - 1; ++i) {
          const double f = s * e[i], b = c * e[i];
          dlartg(g, f, c, s, r);
          if (i != mq) e[i - 1] = r;
          g = d[i] - p;
          r = (d[i + 1] - g) * s + 2.0 * c * b;
          p = s * r;
          d[i] = g + p;
          g = c * r - b;
          wc[i - mq] = c;
          ws[i - mq] = s;
        }
        dlasr_rv(z, mq, l - mq + 1, wc, ws, true);
        d[l] = d[l] - p;
        e[l - 1] = g;
      }
    }
    if (jtot >= nmaxit) return false;
  }
  // selection sort (ascending), swapping eigenvector columns
  for (int ii = 1; ii < n; ++ii) {
    const int i = ii - 1;
    int k = i;
    double p = d[i];
    for (int j = ii; j < n; ++j)
      if (d[j] < p) {
        k = j;
        p = d[j];
      }
    if (k != i) {
      d[k] = d[i];
      d[i] = p;
      for (int r = 0; r < 3; ++r) {
        const double t = z[r][i];
        z[r][i] = z[r][k];
        z[r][k] = t;
      }
    }
  }
  return true;
}

// dsyevd('V', 'L') of a symmetric 3x3 (only the lower triangle a[i][j], i >= j, is read).
// w ascending; v[r][c] = component r of eigenvector c.
SS_HD bool eigh3(const double a_in[3][3], double w[3], double v[3][3]) {
  double a[3][3];
  for (int i = 0; i < 3; ++i)
    for (int j = 0; j < 3; ++j) a[i][j] = a_in[i][j];
  // dsytd2, UPLO='L': reflector H(1) on rows 2..3 of column 1
  const double alpha = a[1][0], x = a[2][0];
  double tau = 0.0, v2 = 0.0, beta = alpha;
  const double xnorm = fabs(x);
  if (xnorm != 0.0) {
    beta = -sgn(dlapy2(alpha, xnorm), alpha);
    tau = (beta - alpha) / beta;
    v2 = x * (1.0 / (alpha - beta));
  }
  double e[2], d[3];
  e[0] = beta;
  if (tau != 0.0) {
    // w = tau * B v (dsymv, lower), B = a[1..2][1..2], v = (1, v2)
    double y0 = 0.0, y1 = 0.0;
    {
      double temp1 = tau * 1.0, temp2 = 0.0;
      y0 += temp1 * a[1][1];
      y1 += temp1 * a[2][1];
      temp2 += a[2][1] * v2;
      y0 += tau * temp2;
      temp1 = tau * v2;
      y1 += temp1 * a[2][2];
    }
    const double alpha2 = -0.5 * tau * (y0 * 1.0 + y1 * v2);
    y0 += alpha2 * 1.0;
    y1 += alpha2 * v2;
    // B -= v w^T + w v^T (dsyr2, lower)
    a[1][1] = a[1][1] + (1.0 * (-y0) + y0 * (-1.0));
    a[2][1] = a[2][1] + (v2 * (-y0) + y1 * (-1.0));
    a[2][2] = a[2][2] + (v2 * (-y1) + y1 * (-v2));
  }
  d[0] = a[0][0];
  // H(2): dlarfg with n = 1 -> tau = 0, e(2) = a(3,2)
  e[1] = a[2][1];
  d[1] = a[1][1];
  d[2] = a[2][2];
  double z[3][3];
  if (!dsteqr3(d, e, z)) return false;
  // dorm2r: Z <- diag(1, H(1)) Z, H(1) = I - tau (1, v2)(1, v2)^T on rows 2..3
  if (tau != 0.0)
    for (int j = 0; j < 3; ++j) {
      const double wj = z[1][j] + z[2][j] * v2;
      z[1][j] = z[1][j] - tau * wj;
      z[2][j] = z[2][j] - tau * v2 * wj;
    }
  for (int i = 0; i < 3; ++i) {
    w[i] = d[i];
    for (int j = 0; j < 3; ++j) v[i][j] = z[i][j];
  }
  return true;
}

}  // namespace lapack3
}  // namespace ss
