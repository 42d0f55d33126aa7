/* conv_oracle.c -- TEST INFRASTRUCTURE ONLY (oracle, never shipped or measured as
 * the product).  Plain-C restatement of the reference's direct-loop 3D
 * convolution kernels, reference pkg/src/voxpar/kernels/_hot.pyx:
 *   conv3d_fwd        :19-41   y[n,co,z,h,x] += w[co,ci,a,b,c] * xpad[n,ci,sd*z+a,sh*h+b,sw*x+c]
 *   conv3d_bwd_data   :44-67   xg[n,ci,sd*z+a,...] += w[co,ci,a,b,c] * u[n,co,z,h,x]
 *   conv3d_bwd_filter :70-93   wg[co,ci,a,b,c] += sum_{z,h,x} u[n,co,..] * xpad[n,ci,..]
 * Per output element the accumulation order is the reference's loop-nest order
 * and the file is compiled with -ffp-contract=off, so results are bit-identical
 * to the reference's Cython build (checked in tests/test_oracle.py).  The only
 * change is OpenMP parallelism over the loop levels whose iterations write
 * disjoint outputs ((n,co) / (n,ci) / (co,ci)); that leaves every element's
 * summation order untouched.  All arrays are C-contiguous NCDHW / OIDHW.
 */
#include <stddef.h>
#include <stdint.h>

#ifdef _OPENMP
#include <omp.h>
#endif

typedef long long ll;

#define DEFINE_KERNELS(T, SUF)                                                                    \
  void vox_conv3d_fwd_##SUF(const T* xpad, ll n, ll cin, ll pd, ll ph, ll pw, const T* w,        \
                            ll cout, ll kd, ll kh, ll kw, ll sd, ll sh, ll sw, T* y, ll od,      \
                            ll oh, ll ow, int threads) {                                         \
    _Pragma("omp parallel for collapse(2) schedule(dynamic) num_threads(threads)")              \
    for (ll nn = 0; nn < n; ++nn)                                                                \
      for (ll co = 0; co < cout; ++co)                                                           \
        for (ll ci = 0; ci < cin; ++ci)                                                          \
          for (ll a = 0; a < kd; ++a)                                                            \
            for (ll b = 0; b < kh; ++b)                                                          \
              for (ll c = 0; c < kw; ++c) {                                                      \
                const T wv = w[(((co * cin + ci) * kd + a) * kh + b) * kw + c];                  \
                for (ll z = 0; z < od; ++z) {                                                    \
                  const ll zz = sd * z + a;                                                      \
                  for (ll h = 0; h < oh; ++h) {                                                  \
                    const ll hh = sh * h + b;                                                    \
                    const T* xr = xpad + (((nn * cin + ci) * pd + zz) * ph + hh) * pw + c;       \
                    T* yr = y + (((nn * cout + co) * od + z) * oh + h) * ow;                      \
                    for (ll x = 0; x < ow; ++x) yr[x] += wv * xr[sw * x];                        \
                  }                                                                              \
                }                                                                                \
              }                                                                                  \
  }                                                                                              \
  void vox_conv3d_bwd_data_##SUF(const T* u, ll n, ll cout, ll od, ll oh, ll ow, const T* w,     \
                                 ll cin, ll kd, ll kh, ll kw, ll sd, ll sh, ll sw, T* xg, ll pd, \
                                 ll ph, ll pw, int threads) {                                    \
    _Pragma("omp parallel for collapse(2) schedule(dynamic) num_threads(threads)")              \
    for (ll nn = 0; nn < n; ++nn)                                                                \
      for (ll ci = 0; ci < cin; ++ci)                                                            \
        for (ll co = 0; co < cout; ++co)                                                         \
          for (ll a = 0; a < kd; ++a)                                                            \
            for (ll b = 0; b < kh; ++b)                                                          \
              for (ll c = 0; c < kw; ++c) {                                                      \
                const T wv = w[(((co * cin + ci) * kd + a) * kh + b) * kw + c];                  \
                for (ll z = 0; z < od; ++z) {                                                    \
                  const ll zz = sd * z + a;                                                      \
                  for (ll h = 0; h < oh; ++h) {                                                  \
                    const ll hh = sh * h + b;                                                    \
                    T* gr = xg + (((nn * cin + ci) * pd + zz) * ph + hh) * pw + c;               \
                    const T* ur = u + (((nn * cout + co) * od + z) * oh + h) * ow;               \
                    for (ll x = 0; x < ow; ++x) gr[sw * x] += wv * ur[x];                        \
                  }                                                                              \
                }                                                                                \
              }                                                                                  \
  }                                                                                              \
  void vox_conv3d_bwd_filter_##SUF(const T* xpad, ll n, ll cin, ll pd, ll ph, ll pw, const T* u, \
                                   ll cout, ll od, ll oh, ll ow, ll kd, ll kh, ll kw, ll sd,     \
                                   ll sh, ll sw, T* wg, int threads) {                           \
    _Pragma("omp parallel for collapse(2) schedule(dynamic) num_threads(threads)")              \
    for (ll co = 0; co < cout; ++co)                                                             \
      for (ll ci = 0; ci < cin; ++ci)                                                            \
        for (ll nn = 0; nn < n; ++nn)                                                            \
          for (ll a = 0; a < kd; ++a)                                                            \
            for (ll b = 0; b < kh; ++b)                                                          \
              for (ll c = 0; c < kw; ++c) {                                                      \
                T s = 0;                                                                         \
                for (ll z = 0; z < od; ++z) {                                                    \
                  const ll zz = sd * z + a;                                                      \
                  for (ll h = 0; h < oh; ++h) {                                                  \
                    const ll hh = sh * h + b;                                                    \
                    const T* ur = u + (((nn * cout + co) * od + z) * oh + h) * ow;               \
                    const T* xr = xpad + (((nn * cin + ci) * pd + zz) * ph + hh) * pw + c;       \
                    for (ll x = 0; x < ow; ++x) s += ur[x] * xr[sw * x];                         \
                  }                                                                              \
                }                                                                                \
                wg[(((co * cin + ci) * kd + a) * kh + b) * kw + c] += s;                         \
              }                                                                                  \
  }

DEFINE_KERNELS(float, f32)
DEFINE_KERNELS(double, f64)
