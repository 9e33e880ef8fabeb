// H-free Legendre transforms for the table-streaming path (T >= 200).
//
// The spectral-transform f_E (the planar template is
// pkg/src/parsdc/problems/swe.py:174-205) needs, besides P, the table
// H_n = (1 - mu^2) dP_n/dmu: the synthesis of U, V uses H on psi and chi, the
// analysis of div / curl uses H on A, B, D.  For the orthonormal P of order m,
//   H_n = a_n P_{n-1} + b_n P_{n+1},  a_n = (n+1) eps_n,  b_n = -n eps_{n+1},
//   eps_n = sqrt((n^2 - m^2) / (4 n^2 - 1))
// (exact; tests/test_oracle_sphere.py checks it on the oracle's tables), so
//   synthesis:  sum_n X_n H_n = sum_k P_k (a_{k+1} X_{k+1} + b_{k-1} X_{k-1})
//   analysis:   sum_j w Y H_n = a_n Yhat_{n-1} + b_n Yhat_{n+1},  Yhat_k = sum_j w Y P_k
// with k running to T+1.  The f_E chain then streams one table instead of two
// and runs 4 + 5 complex P transforms instead of 4 + 2 (synthesis) and
// 4 + 3 (analysis): 9 instead of 13 per f_E.
//
//   k_xsyn_ponly      xsyn records (12 doubles, the producers' format) -> the
//                     P-only operand (8 doubles per P row: U', V', zeta, Phi)
//   k_synthesis_bulk<NB, true>  (legendre_tma.cu) P-only synthesis
//   k_ring (po)       (ring_fft.cu) five folded, weighted products per (m, j)
//   k_analysis_bulk_ponly       (legendre_tma.cu) P analyses to degree T+1
//   k_assemble_ponly  i m factors + the recurrence -> f_E (Phi', zeta, delta)
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <vector>

#include "internal.cuh"

namespace sdcsw {

cudaError_t launch_synthesis_bulk_ponly(const Plan& p, double2* fsyn, const int* mlist, int nm,
                                        int Lp, const double* xsp, int nb, cudaStream_t s,
                                        int* step_counter, const SynDst& sd);
cudaError_t launch_analysis_bulk_ponly(const Plan& p, const Work& w, int nb, cudaStream_t s);
cudaError_t configure_analysis_bulk_ponly();
cudaError_t make_table_map_ponly(Plan& p);

// ---------------------------------------------------------------------------
// operand conversion: one thread per (P row r, state b, column quad of part 0 or
// part 1 order), enumerated in output order so stores coalesce
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_xsyn_ponly(const double* __restrict__ xsyn, int rows,
                                                    int rowsP, int nb,
                                                    const int4* __restrict__ cvt_rows,
                                                    const double2* __restrict__ cvt_ab,
                                                    double* __restrict__ xsp,
                                                    const int* __restrict__ m_part, int sp) {
  SDCSW_PDL_ENTRY();
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)rowsP * nb;
  if (tid >= total) return;
  const int w = nb;
  const int r4 = (int)(tid / (4 * w)), rem = (int)(tid - (long long)r4 * 4 * w);
  const int b = rem >> 2, rr = rem & 3;
  const int r = 4 * r4 + rr;
  const int4 src = cvt_rows[r];  // constant plan data: before the dependency wait
  const double2 ab = cvt_ab[r];
  SDCSW_PDL_WAIT();
  if (m_part != nullptr && m_part[src.w] != sp) return;  // split plan: own wavenumbers only
  const size_t ps = 16 * (size_t)w;  // part stride of both layouts
  double* out = xsp + ((size_t)r4 * 2 * w + b) * 16 + rr * 4;
  double4 p0 = make_double4(0.0, 0.0, 0.0, 0.0), p1 = p0;
  auto rec = [&](int row) { return xsyn + ((size_t)(row >> 2) * 3 * w + b) * 16 + (row & 3) * 4; };
  if (src.x >= 0) {
    const double* x = rec(src.x);
    p0 = *reinterpret_cast<const double4*>(x);       // U_P, V_P
    p1 = *reinterpret_cast<const double4*>(x + ps);  // zeta, Phi
  }
  if (src.z >= 0) {  // a_{k+1} (U_H, V_H)(k+1)
    const double4 h = *reinterpret_cast<const double4*>(rec(src.z) + 2 * ps);
    p0.x = __fma_rn(ab.x, h.x, p0.x);
    p0.y = __fma_rn(ab.x, h.y, p0.y);
    p0.z = __fma_rn(ab.x, h.z, p0.z);
    p0.w = __fma_rn(ab.x, h.w, p0.w);
  }
  if (src.y >= 0) {  // b_{k-1} (U_H, V_H)(k-1)
    const double4 h = *reinterpret_cast<const double4*>(rec(src.y) + 2 * ps);
    p0.x = __fma_rn(ab.y, h.x, p0.x);
    p0.y = __fma_rn(ab.y, h.y, p0.y);
    p0.z = __fma_rn(ab.y, h.z, p0.z);
    p0.w = __fma_rn(ab.y, h.w, p0.w);
  }
  *reinterpret_cast<double4*>(out) = p0;
  *reinterpret_cast<double4*>(out + ps) = p1;
}

// ---------------------------------------------------------------------------
// operand from the states: the same P-only records as k_xsyn_ponly, built from
// nb states u [b][Phi', zeta, delta][C] complex with the producers' rounding
// (write_xsyn_half: U_P = -i sm delta, V_P = -i sm zeta, U_H = sa zeta,
// V_H = -sa delta, (sm, sa) = xscale), so both routes give the same bits.  The
// dSDC stepper on H-free plans keeps its node states and calls this instead of
// writing 12-double records (96 B) that the conversion re-reads.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_prep_ponly(const double2* __restrict__ u, int C, int rowsP,
                                                    int nb, const int4* __restrict__ prep_idx,
                                                    const double2* __restrict__ cvt_ab,
                                                    const double2* __restrict__ xscale,
                                                    double* __restrict__ xsp) {
  SDCSW_PDL_ENTRY();
  const long long tid = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  const long long total = (long long)rowsP * nb;
  if (tid >= total) return;
  const int w = nb;
  const int r4 = (int)(tid / (4 * w)), rem = (int)(tid - (long long)r4 * 4 * w);
  const int b = rem >> 2, rr = rem & 3;
  const int r = 4 * r4 + rr;
  const int4 ix = prep_idx[r];  // constant plan data: before the dependency wait
  const double2 ab = cvt_ab[r];
  const double2 sc0 = ix.x >= 0 ? xscale[ix.x] : make_double2(0.0, 0.0);
  const double sa_lo = ix.y >= 0 ? xscale[ix.y].y : 0.0, sa_hi = ix.z >= 0 ? xscale[ix.z].y : 0.0;
  SDCSW_PDL_WAIT();
  const double2* s = u + (size_t)b * 3 * C;
  const size_t ps = 16 * (size_t)w;
  double* out = xsp + ((size_t)r4 * 2 * w + b) * 16 + rr * 4;
  double4 p0 = make_double4(0.0, 0.0, 0.0, 0.0), p1 = p0;
  if (ix.x >= 0) {
    const double2 phi = s[ix.x], zeta = s[C + ix.x], delta = s[2 * C + ix.x];
    const double sm = sc0.x;
    p0 = make_double4(sm * delta.y, -sm * delta.x, sm * zeta.y, -sm * zeta.x);  // U_P, V_P
    p1 = make_double4(zeta.x, zeta.y, phi.x, phi.y);
  }
  if (ix.z >= 0) {  // a_{k+1} (U_H, V_H)(k+1)
    const double2 z = s[C + ix.z], d = s[2 * C + ix.z];
    p0.x = __fma_rn(ab.x, sa_hi * z.x, p0.x);
    p0.y = __fma_rn(ab.x, sa_hi * z.y, p0.y);
    p0.z = __fma_rn(ab.x, -sa_hi * d.x, p0.z);
    p0.w = __fma_rn(ab.x, -sa_hi * d.y, p0.w);
  }
  if (ix.y >= 0) {  // b_{k-1} (U_H, V_H)(k-1)
    const double2 z = s[C + ix.y], d = s[2 * C + ix.y];
    p0.x = __fma_rn(ab.y, sa_lo * z.x, p0.x);
    p0.y = __fma_rn(ab.y, sa_lo * z.y, p0.y);
    p0.z = __fma_rn(ab.y, -sa_lo * d.x, p0.z);
    p0.w = __fma_rn(ab.y, -sa_lo * d.y, p0.w);
  }
  *reinterpret_cast<double4*>(out) = p0;
  *reinterpret_cast<double4*>(out + ps) = p1;
}

// ---------------------------------------------------------------------------
// assembly: f_E(m, n) from the P analyses at degrees n - 1, n, n + 1
//   Phi'_t = -i m C_n + a_n D_{n-1} + b_n D_{n+1}
//   zeta_t = -i m A_n + a_n B_{n-1} + b_n B_{n+1}
//   delta_t = i m B_n + a_n A_{n-1} + b_n A_{n+1} + lambda_n E_n
// (the same terms as the P/H analysis epilogue, legendre_tma.cu k_analysis_bulk)
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_assemble_ponly(const double* __restrict__ ghat, int C,
                                                        int CP, int nb,
                                                        const int2* __restrict__ asm_pos,
                                                        const double2* __restrict__ asm_ab,
                                                        const double* __restrict__ lam,
                                                        double2* __restrict__ fe,
                                                        const int* __restrict__ idx_list, int n) {
  SDCSW_PDL_ENTRY();
  const int i = blockIdx.x * blockDim.x + threadIdx.x;
  const int b = blockIdx.y;
  if (i >= n || b >= nb) return;
  const int idx = idx_list != nullptr ? idx_list[i] : i;
  const int2 pm = asm_pos[idx];
  const double2 ab = asm_ab[idx];
  const double l = lam[idx];
  SDCSW_PDL_WAIT();
  const double2* g = reinterpret_cast<const double2*>(ghat + ((size_t)b * CP + pm.x) * kGhat);
  const double dm = (double)pm.y;
  // slots: 0 A, 1 B, 2 C, 3 D, 4 E; the n - 1 entry exists unless n = m (a_m = 0)
  const bool lo = ab.x != 0.0;
  const double2 A0 = g[0], B0 = g[1], C0 = g[2], E0 = g[4];
  const double2 Ap = g[kSlotsP + 0], Bp = g[kSlotsP + 1], Dp = g[kSlotsP + 3];
  const double2 Am = lo ? g[-kSlotsP + 0] : make_double2(0.0, 0.0);
  const double2 Bm = lo ? g[-kSlotsP + 1] : make_double2(0.0, 0.0);
  const double2 Dm = lo ? g[-kSlotsP + 3] : make_double2(0.0, 0.0);
  auto rec = [&](double2 m1, double2 p1) {  // a_n X_{n-1} + b_n X_{n+1}
    return make_double2(__fma_rn(ab.x, m1.x, ab.y * p1.x), __fma_rn(ab.x, m1.y, ab.y * p1.y));
  };
  const double2 hd = rec(Dm, Dp), hb = rec(Bm, Bp), ha = rec(Am, Ap);
  double2 phi = make_double2(dm * C0.y + hd.x, -dm * C0.x + hd.y);
  double2 zeta = make_double2(dm * A0.y + hb.x, -dm * A0.x + hb.y);
  double2 delta = make_double2(__fma_rn(l, E0.x, -dm * B0.y + ha.x), __fma_rn(l, E0.y, dm * B0.x + ha.y));
  if (pm.y == 0) phi.y = zeta.y = delta.y = 0.0;
  double2* dst = fe + (size_t)b * 3 * C;
  dst[idx] = phi;
  dst[C + idx] = zeta;
  dst[2 * C + idx] = delta;
}

cudaError_t launch_synthesis_ponly(const Plan& p, double2* fsyn, const int* mlist, int nm, int Lp,
                                   double* xsp, const double* xsyn, int nb, cudaStream_t s,
                                   int* step_counter, const SynDst& sd) {
  const long long total = (long long)p.rowsP * nb;
  const bool own = p.own_idx != nullptr;
  cudaError_t e = launch_k(k_xsyn_ponly, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, s, xsyn,
                           p.rows, p.rowsP, nb, p.cvt_rows, p.cvt_ab, xsp,
                           own ? (const int*)p.m_part : nullptr, p.split_sp);
  if (e != cudaSuccess) return e;
  return launch_synthesis_bulk_ponly(p, fsyn, mlist, nm, Lp, xsp, nb, s, step_counter, sd);
}

cudaError_t f_expl_states_ponly(const Plan& p, const Work& w, const double2* u, double2* fe, int nb,
                                cudaStream_t s, int* step_counter) {
  if (!ponly_on(p) || p.own_idx != nullptr || w.xsp == nullptr) return cudaErrorInvalidValue;
  const long long total = (long long)p.rowsP * nb;
  cudaError_t e = launch_k(k_prep_ponly, dim3((unsigned)((total + 255) / 256)), dim3(256), 0, s, u,
                           p.C, p.rowsP, nb, p.prep_idx, p.cvt_ab, p.xscale, w.xsp);
  if (e == cudaSuccess)
    e = launch_synthesis_bulk_ponly(p, w.fsyn, nullptr, p.T + 1, p.T + 1, w.xsp, nb, s, step_counter,
                                    SynDst{});
  if (e == cudaSuccess) e = launch_ring(p, w, nb, s);
  if (e == cudaSuccess) e = launch_analysis_ponly(p, w, fe, nb, s);
  return e;
}

cudaError_t f_expl_operand_ponly(const Plan& p, const Work& w, const double* xsp, double2* fe, int nb,
                                 cudaStream_t s) {
  if (!ponly_on(p) || p.own_idx != nullptr || xsp == nullptr) return cudaErrorInvalidValue;
  cudaError_t e = launch_synthesis_bulk_ponly(p, w.fsyn, nullptr, p.T + 1, p.T + 1, xsp, nb, s,
                                              nullptr, SynDst{});
  if (e == cudaSuccess) e = launch_ring(p, w, nb, s);
  if (e == cudaSuccess) e = launch_analysis_ponly(p, w, fe, nb, s);
  return e;
}

cudaError_t launch_analysis_ponly(const Plan& p, const Work& w, double2* fe, int nb, cudaStream_t s) {
  cudaError_t e = launch_analysis_bulk_ponly(p, w, nb, s);
  if (e != cudaSuccess) return e;
  const bool own = p.own_idx != nullptr;  // split plan: own coefficients only
  const int n = own ? p.n_own_idx : p.C;
  if (n < 1) return cudaSuccess;
  return launch_k(k_assemble_ponly, dim3((n + 255) / 256, nb), dim3(256), 0, s,
                  (const double*)w.ghat, p.C, p.CP, nb, p.asm_pos, p.asm_ab, p.lam, fe,
                  own ? (const int*)p.own_idx : nullptr, n);
}

// ---------------------------------------------------------------------------
// plan setup: extended P table (degree T+1 from the three-term recurrence
// mu P_n = eps_{n+1} P_{n+1} + eps_n P_{n-1}, in long double), index maps
// ---------------------------------------------------------------------------
static long double eps_l(int n, int m) {
  if (n <= m) return 0.0L;  // eps_m^m = 0
  return sqrtl(((long double)n * n - (long double)m * m) / (4.0L * n * n - 1.0L));
}

void ponly_free(Plan& p) {
  void* ptrs[] = {p.ptabP, p.ptabP_s, p.rowoffP, p.n_evenP, p.rowP_n, p.moffP, p.cvt_rows, p.prep_idx,
                  p.coef_prow,
                  p.cvt_ab, p.asm_pos, p.asm_ab, p.anal_workP, p.own_workP, p.xsynP, p.ghat};
  for (void* q : ptrs)
    if (q) dev_free(q);
  p.ptabP = p.ptabP_s = nullptr;
  p.rowoffP = p.n_evenP = p.rowP_n = p.moffP = p.anal_workP = p.own_workP = nullptr;
  p.cvt_rows = p.prep_idx = p.coef_prow = nullptr;
  p.cvt_ab = p.asm_ab = nullptr;
  p.asm_pos = nullptr;
  p.xsynP = p.ghat = nullptr;
}

template <typename T>
static cudaError_t up(T** dst, const std::vector<T>& v, size_t pad = 0) {
  cudaError_t e = dev_alloc(dst, (v.size() + pad) * sizeof(T));
  if (e != cudaSuccess) return e;
  if (pad) e = cudaMemset(*dst + v.size(), 0, pad * sizeof(T));
  if (e == cudaSuccess && !v.empty())
    e = cudaMemcpy(*dst, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice);
  return e;
}

cudaError_t ponly_setup(Plan& p, const double* ptab, const int* rowoff, const int* row_n,
                        const double* mu_north) {
  const int T = p.T, J = p.J, C = p.C;
  if (J % 32 != 0) return cudaErrorNotSupported;  // bulk synthesis tiles
  std::vector<int> moff(T + 2), xrow(C, -1);
  for (int m = 0; m <= T + 1; ++m) moff[m] = m * (T + 1) - m * (m - 1) / 2;
  for (int m = 0; m <= T; ++m)
    for (int r = rowoff[m]; r < rowoff[m + 1]; ++r)
      if (row_n[r] >= 0) xrow[moff[m] + row_n[r] - m] = r;
  auto xr = [&](int m, int n) { return (n < m || n > T) ? -1 : xrow[moff[m] + n - m]; };
  // extended rows: degrees m..T+1 per m, parity-sorted, each class padded to 8
  std::vector<int> rowoffP(T + 2), n_evenP(T + 1), rowP_n, moffP(T + 2);
  rowoffP[0] = 0;
  moffP[0] = 0;
  for (int m = 0; m <= T; ++m) {
    const int len = T + 2 - m, ne = (len + 1) / 2, no = len / 2;
    const int ne8 = (ne + kRowPad - 1) / kRowPad * kRowPad, no8 = (no + kRowPad - 1) / kRowPad * kRowPad;
    n_evenP[m] = ne8;
    for (int i = 0; i < ne8; ++i) rowP_n.push_back(i < ne ? m + 2 * i : -1);
    for (int i = 0; i < no8; ++i) rowP_n.push_back(i < no ? m + 1 + 2 * i : -1);
    rowoffP[m + 1] = rowoffP[m] + ne8 + no8;
    moffP[m + 1] = moffP[m] + len;
  }
  const int rowsP = rowoffP[T + 1], CP = moffP[T + 1];
  std::vector<double> tabP((size_t)rowsP * J, 0.0), tabS((size_t)rowsP * J, 0.0);
  std::vector<int4> cvt(rowsP), pidx(rowsP);
  std::vector<double2> cab(rowsP);
  for (int m = 0; m <= T; ++m)
    for (int r = rowoffP[m]; r < rowoffP[m + 1]; ++r) {
      const int k = rowP_n[r];
      cvt[r] = make_int4(-1, -1, -1, m);
      pidx[r] = make_int4(-1, -1, -1, m);
      cab[r] = make_double2(0.0, 0.0);
      if (k < 0) continue;
      double* dst = tabP.data() + (size_t)r * J;
      if (k <= T) {
        std::memcpy(dst, ptab + (size_t)xr(m, k) * J, J * sizeof(double));
      } else {  // P_{T+1} = (mu P_T - eps_T P_{T-1}) / eps_{T+1}
        const double* pT = ptab + (size_t)xr(m, T) * J;
        const double* pT1 = T - 1 >= m ? ptab + (size_t)xr(m, T - 1) * J : nullptr;
        const long double eT = eps_l(T, m), eT1 = eps_l(T + 1, m);
        for (int j = 0; j < J; ++j) {
          long double v = (long double)mu_north[j] * pT[j];
          if (pT1) v -= eT * pT1[j];
          dst[j] = (double)(v / eT1);
        }
      }
      cvt[r] = make_int4(xr(m, k), k - 1 >= m ? xr(m, k - 1) : -1, xr(m, k + 1), m);
      auto ci = [&](int n) { return (n < m || n > T) ? -1 : moff[m] + n - m; };
      pidx[r] = make_int4(ci(k), ci(k - 1), ci(k + 1), m);
      // a_{k+1} = (k + 2) eps_{k+1}, b_{k-1} = -(k - 1) eps_k
      cab[r] = make_double2((double)((k + 2) * eps_l(k + 1, m)), (double)(-(k - 1) * eps_l(k, m)));
    }
  for (int r = 0; r < rowsP; ++r)
    for (int j = 0; j < J; ++j)
      tabS[(((size_t)(r / 4) * (J / 8) + j / 8) * 8 + j % 8) * 4 + r % 4] = tabP[(size_t)r * J + j];
  std::vector<int2> apos(C);
  std::vector<double2> aab(C);
  std::vector<int4> cprow(C);
  for (int m = 0; m <= T; ++m)
    for (int r = rowoffP[m]; r < rowoffP[m + 1]; ++r) {
      const int k = rowP_n[r];
      if (k < 0) continue;
      if (k <= T) {
        int4& c = cprow[moff[m] + k - m];
        c.x = r;
        c.z = k > m ? 1 : 0;
        c.w = k < T ? 1 : 0;
        if (k < T) c.y = -1;
      } else {
        cprow[moff[m] + T - m].y = r;  // the extra degree-(T+1) row, written by (m, T)
      }
    }
  for (int m = 0; m <= T; ++m)
    for (int n = m; n <= T; ++n) {
      const int idx = moff[m] + n - m;
      apos[idx] = make_int2(moffP[m] + n - m, m);
      aab[idx] = make_double2((double)((n + 1) * eps_l(n, m)), (double)(-n * eps_l(n + 1, m)));
    }
  std::vector<int> work;
  for (int m = 0; m <= T; ++m) {
    const int rows = rowoffP[m + 1] - rowoffP[m];
    for (int rb = 0; rb * 4 * kRowsPerWarp < rows; ++rb) work.push_back((m << 16) | rb);
  }
  p.rowsP = rowsP;
  p.CP = CP;
  p.n_anal_workP = (int)work.size();
  cudaError_t e;
  if ((e = up(&p.ptabP, tabP, (size_t)16 * J)) != cudaSuccess ||
      (e = up(&p.ptabP_s, tabS, (size_t)16 * J)) != cudaSuccess ||
      (e = up(&p.rowoffP, rowoffP)) != cudaSuccess || (e = up(&p.n_evenP, n_evenP)) != cudaSuccess ||
      (e = up(&p.rowP_n, rowP_n, 16)) != cudaSuccess || (e = up(&p.moffP, moffP)) != cudaSuccess ||
      (e = up(&p.cvt_rows, cvt)) != cudaSuccess || (e = up(&p.cvt_ab, cab)) != cudaSuccess ||
      (e = up(&p.prep_idx, pidx)) != cudaSuccess || (e = up(&p.coef_prow, cprow)) != cudaSuccess ||
      (e = up(&p.asm_pos, apos)) != cudaSuccess || (e = up(&p.asm_ab, aab)) != cudaSuccess ||
      (e = up(&p.anal_workP, work)) != cudaSuccess ||
      (e = dev_alloc(&p.xsynP, (size_t)p.max_batch * rowsP * kXsynP * sizeof(double))) != cudaSuccess ||
      // padding rows must read as zero (k_sweep_nodes_po writes valid rows only)
      (e = cudaMemset(p.xsynP, 0, (size_t)p.max_batch * rowsP * kXsynP * sizeof(double))) != cudaSuccess ||
      (e = dev_alloc(&p.ghat, (size_t)p.max_batch * CP * kGhat * sizeof(double))) != cudaSuccess ||
      (e = configure_analysis_bulk_ponly()) != cudaSuccess || (e = make_table_map_ponly(p)) != cudaSuccess) {
    ponly_free(p);
    return e;
  }
  return cudaSuccess;
}

}  // namespace sdcsw
