// Node-to-node sweep kernels in spectral space: quadrature Q.F, the
// MIN-SR-FLEX diagonal right-hand side, the per-degree 2x2 implicit solve and
// f_I of the result, for all collocation nodes in one pass over the state.
//
// Every operation is an explicitly rounded IEEE op (__dmul_rn, __dadd_rn, ...;
// never contracted into FMA) in the order numpy evaluates the reference
// expressions, so results are bit-identical to the reference / oracle given
// identical inputs:
//   diagonal_sweep phase one      pkg/src/parsdc/integrators.py:268-277
//   _refresh_node solve + f_impl  integrators.py:233-246 (f_expl is separate)
//   _final_node_solve             integrators.py:291-311
//   serial_sweep                  integrators.py:183-230
//   planar solve / f_impl         problems/swe.py:157-172 with k^2 -> n(n+1)/a^2
// One thread owns one (m, n) coefficient index and its three fields; memory
// traffic is (1 + 2M) state reads and 2M state writes per sweep.
#include <climits>
#include <cstdlib>

#include "node_math.cuh"

namespace sdcsw {

// ---------------------------------------------------------------------------
// diagonal sweep, nodes [lo, lo+count): grid (ceil(2C/256), count)
// coef layout per node m: w[0..M-1], wd, alpha, a_phi, a2_phi  (stride M+4)
// ---------------------------------------------------------------------------
// grid (ceil(2C/256), count, members); member z reads u0 + z S, fe + z fe_mstride,
// fi + z fi_mstride and writes batch entry z * count + q of the outputs.
__global__ void __launch_bounds__(256) k_sweep_nodes(
    int C2, int M, int lo, NodeArgs cf, const double* __restrict__ u0,
    const double* __restrict__ fe, long long fe_stride, const double* __restrict__ fi,
    long long fi_stride, int first, double phibar, const double* __restrict__ lamv,
    double* __restrict__ u_out, double* fi_out, const double2* __restrict__ xscale,
    const int* __restrict__ idx_row, double* __restrict__ xsyn, long long fe_mstride,
    long long fi_mstride, int rows, int chunk, const int* __restrict__ idx_list, int n_list,
    PeerWait pw) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  const long long par = peer_wait(pw);  // node-parallel: the latest exchange's parity
  fe += par;
  fi += par;
  int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx_list != nullptr) {  // spectral split: own coefficients only
    if (e >= 2 * n_list) return;
    e = 2 * idx_list[e >> 1] + (e & 1);
  }
  if (e >= C2) return;
  const int z = blockIdx.z;
  u0 += (size_t)z * 3 * C2;
  fe += z * fe_mstride;
  fi += z * fi_mstride;
  const int q = blockIdx.y, m = lo + q;
  const int ob = z * gridDim.y + q;  // output batch entry
  const double lam = lamv[e >> 1];
  const Tri a0 = load_tri(u0, C2, e);
  const Tri fi0 = f_impl_tri(a0, phibar, lam);
  const double* c = cf.v + m * (M + 4);
  Tri b = a0, fim = fi0;
  for (int j = 0; j < M; ++j) {
    const Tri ej = load_tri(fe + j * fe_stride, C2, e);
    const Tri ij = first ? fi0 : load_tri(fi + j * fi_stride, C2, e);
    b = axpy_tri(b, c[j], add_tri(ej, ij));
    if (j == m) fim = ij;
  }
  b = axmy_tri(b, c[M], fim);
  const Tri u = solve_tri(b, c[M + 1], c[M + 2], c[M + 3], lam);
  if (u_out != nullptr) store_tri(u_out + (size_t)ob * 3 * C2, C2, e, u);
  store_tri(fi_out + (size_t)ob * 3 * C2, C2, e, f_impl_tri(u, phibar, lam));
  if (xsyn != nullptr) {  // synthesis B operand of the f_E that follows, in batch chunks
    const int nbt = gridDim.y * gridDim.z, ch = chunk > 0 ? chunk : nbt;
    const int cb = ob / ch, w = nbt - cb * ch < ch ? nbt - cb * ch : ch;
    write_xsyn_half(xsyn + (size_t)cb * rows * ch * kXsyn + xsyn_off(idx_row[e >> 1], ob - cb * ch, w),
                    16 * (size_t)w, e & 1, u.phi, u.zeta, u.delta, xscale[e >> 1]);
  }
}

// ---------------------------------------------------------------------------
// Collocation-residual norms, fused into the sweep kernel (opt-in): per node
// and field, ||u0 + sum_j w_mj (fe_j + fi_j) - u_prev_m||_2 over the stored
// complex coefficients.  Deterministic: a fixed-order block tree, per-block
// partials, and the last block to finish sums the partials in block order
// (then re-arms the counter for the next call).
// ---------------------------------------------------------------------------
__device__ void resid_block(const ResidArgs& ra, const double (*ss)[3], int count) {
  __shared__ double red[256];
  __shared__ bool last;
  const int nv = count * 3;
  for (int v = 0; v < nv; ++v) {
    red[threadIdx.x] = ss != nullptr ? ss[v / 3][v % 3] : 0.0;
    __syncthreads();
    for (int h = 128; h > 0; h >>= 1) {
      if (threadIdx.x < h) red[threadIdx.x] += red[threadIdx.x + h];
      __syncthreads();
    }
    if (threadIdx.x == 0) ra.part[(size_t)v * gridDim.x + blockIdx.x] = red[0];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(ra.count, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  if (threadIdx.x < nv) {
    double acc = 0.0;
    const volatile double* pv = ra.part + (size_t)threadIdx.x * gridDim.x;
    for (unsigned b = 0; b < gridDim.x; ++b) acc += pv[b];
    ra.out[threadIdx.x] = sqrt(acc);
  }
  if (threadIdx.x == 0) *ra.count = 0u;
}

// ---------------------------------------------------------------------------
// The same node updates with one thread per coefficient (both components,
// 16-byte accesses) for all nodes of the block [lo, lo + count): u0 and every
// fe_j, fi_j are read once (instead of once per node) and the synthesis
// operand is written in whole 32-byte chunks - the sweep is HBM-bound at large
// T.  Same rounded arithmetic as k_sweep_nodes (bit-identical).
// M <= kFuseMaxNodes.
// ---------------------------------------------------------------------------
template <bool RES>  // RES: fused collocation-residual norms (resid_block)
__global__ void __launch_bounds__(256) k_sweep_nodes_all(
    int C, int M, int lo, int count, NodeArgs cf, const double* __restrict__ u0,
    const double* __restrict__ fe, long long fe_stride, const double* __restrict__ fi,
    long long fi_stride, int first, double phibar, const double* __restrict__ lamv,
    double* __restrict__ u_out, double* fi_out, const double2* __restrict__ xscale,
    const int* __restrict__ idx_row, double* __restrict__ xsyn, long long fe_mstride,
    long long fi_mstride, int rows, int chunk, const int* __restrict__ idx_list, int n_list,
    PeerWait pw, ResidArgs ra) {
  SDCSW_PDL_ENTRY();
  constexpr int MX = kFuseMaxNodes;
  const long long par = peer_wait(pw);  // node-parallel: the latest exchange's parity
  fe += par;
  fi += par;
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx_list != nullptr) {  // spectral split: own coefficients only (no residual)
    if (idx >= n_list) return;
    idx = idx_list[idx];
  }
  // with RES every thread of the block must reach the one resid_block call (it holds
  // block barriers), so tail threads stay converged with zero contributions
  const bool active = idx < C;
  if constexpr (!RES) {
    if (!active) return;
  }
  double ss[RES ? MX : 1][3] = {};  // residual: squared norms per (node, field) of this coefficient
  if (active) {
    const double lam = lamv[idx];
    const double2 sc = xscale != nullptr ? xscale[idx] : make_double2(0.0, 0.0);
    const int row = xsyn != nullptr ? idx_row[idx] : 0;
    SDCSW_PDL_WAIT();
    const int z = blockIdx.z;
    const int C2 = 2 * C;
    u0 += (size_t)z * 3 * C2;
    fe += z * fe_mstride;
    fi += z * fi_mstride;
    Tri a0r, a0i;
    load_tri2(u0, C, idx, a0r, a0i);
    const Tri f0r = f_impl_tri(a0r, phibar, lam), f0i = f_impl_tri(a0i, phibar, lam);
    Tri Fr[MX], Fi[MX], Ir[MX], Ii[MX];
#pragma unroll
    for (int j = 0; j < MX; ++j)
      if (j < M) {
        load_tri2(fe + j * fe_stride, C, idx, Fr[j], Fi[j]);
        if (first) {
          Ir[j] = f0r;
          Ii[j] = f0i;
        } else {
          load_tri2(fi + j * fi_stride, C, idx, Ir[j], Ii[j]);
        }
      }
    const int nbt = count * gridDim.z, ch = chunk > 0 ? chunk : nbt;
    for (int q = 0; q < count; ++q) {
      const int m = lo + q;
      const int ob = z * count + q;  // output batch entry
      const double* c = cf.v + m * (M + 4);
      Tri br = a0r, bi = a0i, fmr = f0r, fmi = f0i;
#pragma unroll
      for (int j = 0; j < MX; ++j)
        if (j < M) {
          br = axpy_tri(br, c[j], add_tri(Fr[j], Ir[j]));
          bi = axpy_tri(bi, c[j], add_tri(Fi[j], Ii[j]));
          if (j == m) {
            fmr = Ir[j];
            fmi = Ii[j];
          }
        }
      if constexpr (RES) {  // collocation residual of the previous iterate at node m:
        // u0 + sum_j w_mj F_j (the quadrature just formed) - u_prev_m
        Tri pr, pi;
        load_tri2(ra.u_prev + (size_t)q * 3 * C2, C, idx, pr, pi);
        const double d[3][2] = {{br.phi - pr.phi, bi.phi - pi.phi},
                                {br.zeta - pr.zeta, bi.zeta - pi.zeta},
                                {br.delta - pr.delta, bi.delta - pi.delta}};
#pragma unroll
        for (int f = 0; f < 3; ++f) ss[q][f] = d[f][0] * d[f][0] + d[f][1] * d[f][1];
      }
      br = axmy_tri(br, c[M], fmr);
      bi = axmy_tri(bi, c[M], fmi);
      const Tri ur = solve_tri(br, c[M + 1], c[M + 2], c[M + 3], lam);
      const Tri ui = solve_tri(bi, c[M + 1], c[M + 2], c[M + 3], lam);
      if (u_out != nullptr) store_tri2(u_out + (size_t)ob * 3 * C2, C, idx, ur, ui);
      store_tri2(fi_out + (size_t)ob * 3 * C2, C, idx, f_impl_tri(ur, phibar, lam),
                 f_impl_tri(ui, phibar, lam));
      if (xsyn != nullptr) {
        const int cb = ob / ch, w = nbt - cb * ch < ch ? nbt - cb * ch : ch;
        write_xsyn_full(xsyn + (size_t)cb * rows * ch * kXsyn + xsyn_off(row, ob - cb * ch, w),
                        16 * (size_t)w, ur, ui, sc);
      }
    }
  } else {
    SDCSW_PDL_WAIT();
  }
  if constexpr (RES) resid_block(ra, ss, count);
}

// ---------------------------------------------------------------------------
// H-free dSDC sweep (legendre_ponly.cu): the node updates of k_sweep_nodes_all
// (same rounded arithmetic, bit-identical f_I) writing, instead of the node
// states, the P-only synthesis operand of the new states - the records
// k_prep_ponly would build from them, bit for bit.  The record of degree n needs
// U_H, V_H of degrees n -+ 1, which adjacent threads hold (coefficients of one m
// are consecutive): each warp owns 30 coefficients and its lanes 0 and 31 are a
// halo (they update the neighbouring warps' first / last coefficient, store
// nothing), and the neighbours' values arrive by warp shuffles.  M <= kFuseMaxNodes.
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_sweep_nodes_po(
    int C, int M, int lo, int count, NodeArgs cf, const double* __restrict__ u0,
    const double* __restrict__ fe, long long fe_stride, const double* __restrict__ fi,
    long long fi_stride, int first, double phibar, const double* __restrict__ lamv,
    double* fi_out, const double2* __restrict__ xscale, const int4* __restrict__ coef_prow,
    const double2* __restrict__ cvt_ab, double* __restrict__ xsp, long long fe_mstride,
    long long fi_mstride) {
  SDCSW_PDL_ENTRY();
  constexpr int MX = kFuseMaxNodes;
  const int lane = threadIdx.x & 31;
  const int gw = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int idx = gw * 30 + lane - 1;
  const bool own = lane >= 1 && lane <= 30 && idx < C;
  const int ic = idx < 0 ? 0 : (idx >= C ? C - 1 : idx);  // halo / tail lanes compute a clamped one
  // constant plan data before the dependency wait
  const double lam = lamv[ic];
  const double2 sc = xscale[ic];
  const int4 pr = coef_prow[ic];
  const double2 ab = cvt_ab[pr.x];
  const double bx = pr.y >= 0 ? cvt_ab[pr.y].y : 0.0;  // b_T of the degree-(T+1) row
  SDCSW_PDL_WAIT();
  const int z = blockIdx.z;
  const int C2 = 2 * C;
  u0 += (size_t)z * 3 * C2;
  fe += z * fe_mstride;
  fi += z * fi_mstride;
  Tri a0r, a0i;
  load_tri2(u0, C, ic, a0r, a0i);
  const Tri f0r = f_impl_tri(a0r, phibar, lam), f0i = f_impl_tri(a0i, phibar, lam);
  Tri Fr[MX], Fi[MX], Ir[MX], Ii[MX];
#pragma unroll
  for (int j = 0; j < MX; ++j)
    if (j < M) {
      load_tri2(fe + j * fe_stride, C, ic, Fr[j], Fi[j]);
      if (first) {
        Ir[j] = f0r;
        Ii[j] = f0i;
      } else {
        load_tri2(fi + j * fi_stride, C, ic, Ir[j], Ii[j]);
      }
    }
  const int nbt = count * gridDim.z;       // operand batch of the chain
  const size_t ps = 16 * (size_t)nbt;      // part stride of the P-only records
  auto rec_of = [&](int r, int b) { return xsp + ((size_t)(r >> 2) * 2 * nbt + b) * 16 + (r & 3) * 4; };
  for (int q = 0; q < count; ++q) {
    const int m = lo + q;
    const int ob = z * count + q;  // output batch entry
    const double* c = cf.v + m * (M + 4);
    Tri br = a0r, bi = a0i, fmr = f0r, fmi = f0i;
#pragma unroll
    for (int j = 0; j < MX; ++j)
      if (j < M) {
        br = axpy_tri(br, c[j], add_tri(Fr[j], Ir[j]));
        bi = axpy_tri(bi, c[j], add_tri(Fi[j], Ii[j]));
        if (j == m) {
          fmr = Ir[j];
          fmi = Ii[j];
        }
      }
    br = axmy_tri(br, c[M], fmr);
    bi = axmy_tri(bi, c[M], fmi);
    const Tri ur = solve_tri(br, c[M + 1], c[M + 2], c[M + 3], lam);
    const Tri ui = solve_tri(bi, c[M + 1], c[M + 2], c[M + 3], lam);
    if (own)
      store_tri2(fi_out + (size_t)ob * 3 * C2, C, idx, f_impl_tri(ur, phibar, lam),
                 f_impl_tri(ui, phibar, lam));
    // U_H = sa zeta, V_H = -sa delta (the producers' rounded products); neighbours by shuffle
    const double sa = sc.y, sm = sc.x;
    const double uhr = sa * ur.zeta, uhi = sa * ui.zeta, vhr = -sa * ur.delta, vhi = -sa * ui.delta;
    const double hur = __shfl_down_sync(0xffffffffu, uhr, 1), hui = __shfl_down_sync(0xffffffffu, uhi, 1);
    const double hvr = __shfl_down_sync(0xffffffffu, vhr, 1), hvi = __shfl_down_sync(0xffffffffu, vhi, 1);
    const double lur = __shfl_up_sync(0xffffffffu, uhr, 1), lui = __shfl_up_sync(0xffffffffu, uhi, 1);
    const double lvr = __shfl_up_sync(0xffffffffu, vhr, 1), lvi = __shfl_up_sync(0xffffffffu, vhi, 1);
    if (own) {
      double4 p0 = make_double4(sm * ui.delta, -sm * ur.delta, sm * ui.zeta, -sm * ur.zeta);  // U_P, V_P
      if (pr.w) {  // a_{n+1} (U_H, V_H)(n+1)
        p0.x = __fma_rn(ab.x, hur, p0.x);
        p0.y = __fma_rn(ab.x, hui, p0.y);
        p0.z = __fma_rn(ab.x, hvr, p0.z);
        p0.w = __fma_rn(ab.x, hvi, p0.w);
      }
      if (pr.z) {  // b_{n-1} (U_H, V_H)(n-1)
        p0.x = __fma_rn(ab.y, lur, p0.x);
        p0.y = __fma_rn(ab.y, lui, p0.y);
        p0.z = __fma_rn(ab.y, lvr, p0.z);
        p0.w = __fma_rn(ab.y, lvi, p0.w);
      }
      double* r0 = rec_of(pr.x, ob);
      *reinterpret_cast<double4*>(r0) = p0;
      *reinterpret_cast<double4*>(r0 + ps) = make_double4(ur.zeta, ui.zeta, ur.phi, ui.phi);
      if (pr.y >= 0) {  // n = T: the record of degree T+1 is b_T (U_H, V_H)(T)
        double* r1 = rec_of(pr.y, ob);
        *reinterpret_cast<double4*>(r1) = make_double4(__fma_rn(bx, uhr, 0.0), __fma_rn(bx, uhi, 0.0),
                                                       __fma_rn(bx, vhr, 0.0), __fma_rn(bx, vhi, 0.0));
        *reinterpret_cast<double4*>(r1 + ps) = make_double4(0.0, 0.0, 0.0, 0.0);
      }
    }
  }
}

// closing last-node solve, one thread per coefficient (both components)
__global__ void __launch_bounds__(256) k_final_node_c(
    int C, int M, NodeArgs cf, const double* __restrict__ u0, const double* __restrict__ fe,
    long long fe_stride, const double* __restrict__ fi, long long fi_stride, int first,
    double phibar, const double* __restrict__ lamv, double* u_out, int* diverged,
    const int* step_counter, const double2* __restrict__ xscale, const int* __restrict__ idx_row,
    double* __restrict__ xsyn, long long fe_mstride, long long fi_mstride, int rows, int chunk,
    const int* __restrict__ idx_list, int n_list, PeerWait pw) {
  SDCSW_PDL_ENTRY();
  const long long par = peer_wait(pw);  // node-parallel: the latest exchange's parity
  fe += par;
  fi += par;
  int idx = blockIdx.x * blockDim.x + threadIdx.x;
  if (idx_list != nullptr) {
    if (idx >= n_list) return;
    idx = idx_list[idx];
  }
  if (idx >= C) return;
  const double lam = lamv[idx];
  const double2 sc = xsyn != nullptr ? xscale[idx] : make_double2(0.0, 0.0);
  const int row = xsyn != nullptr ? idx_row[idx] : 0;
  SDCSW_PDL_WAIT();
  const int z = blockIdx.z;  // ensemble member
  const int C2 = 2 * C;
  u0 += (size_t)z * 3 * C2;
  u_out += (size_t)z * 3 * C2;
  fe += z * fe_mstride;
  fi += z * fi_mstride;
  Tri a0r, a0i;
  load_tri2(u0, C, idx, a0r, a0i);
  const Tri f0r = f_impl_tri(a0r, phibar, lam), f0i = f_impl_tri(a0i, phibar, lam);
  const double* c = cf.v;
  Tri br = a0r, bi = a0i, flr = f0r, fli = f0i;
  if (M <= kFuseMaxNodes) {
    // every load in flight before the first use (HBM-bound at large T)
    constexpr int MX = kFuseMaxNodes;
    Tri er[MX], ei[MX], ir[MX], ii[MX];
#pragma unroll
    for (int j = 0; j < MX; ++j)
      if (j < M) {
        load_tri2(fe + j * fe_stride, C, idx, er[j], ei[j]);
        ir[j] = f0r;
        ii[j] = f0i;
        if (!first) load_tri2(fi + j * fi_stride, C, idx, ir[j], ii[j]);
      }
#pragma unroll
    for (int j = 0; j < MX; ++j)
      if (j < M) {
        br = axpy_tri(axpy_tri(br, c[j], er[j]), c[j], ir[j]);
        bi = axpy_tri(axpy_tri(bi, c[j], ei[j]), c[j], ii[j]);
        if (j == M - 1) {
          flr = ir[j];
          fli = ii[j];
        }
      }
  } else {
    for (int j = 0; j < M; ++j) {
      Tri er, ei, ir = f0r, ii = f0i;
      load_tri2(fe + j * fe_stride, C, idx, er, ei);
      if (!first) load_tri2(fi + j * fi_stride, C, idx, ir, ii);
      br = axpy_tri(axpy_tri(br, c[j], er), c[j], ir);
      bi = axpy_tri(axpy_tri(bi, c[j], ei), c[j], ii);
      if (j == M - 1) {
        flr = ir;
        fli = ii;
      }
    }
  }
  br = axmy_tri(br, c[M], flr);
  bi = axmy_tri(bi, c[M], fli);
  const Tri ur = solve_tri(br, c[M + 1], c[M + 2], c[M + 3], lam);
  const Tri ui = solve_tri(bi, c[M + 1], c[M + 2], c[M + 3], lam);
  store_tri2(u_out, C, idx, ur, ui);
  if (diverged != nullptr && !(finite_tri(ur) && finite_tri(ui)))
    atomicMin(diverged, step_counter ? *step_counter : 1);
  if (xsyn != nullptr) {  // B operand of the next step's f_E(u0) (batch = members, chunked)
    const int nbt = gridDim.z, ch = chunk > 0 ? chunk : nbt;
    const int cb = z / ch, w = nbt - cb * ch < ch ? nbt - cb * ch : ch;
    write_xsyn_full(xsyn + (size_t)cb * rows * ch * kXsyn + xsyn_off(row, z - cb * ch, w),
                    16 * (size_t)w, ur, ui, sc);
  }
}

// ---------------------------------------------------------------------------
// serial sweep pieces
// ---------------------------------------------------------------------------
// quad_m = u0 + sum_j (w_mj fe_j + w_mj fi_j), grid (ceil(2C/256), M)  (integrators.py:198-205)
__global__ void __launch_bounds__(256) k_serial_quad(
    int C2, int M, NodeArgs cf, const double* __restrict__ u0, const double* __restrict__ fe,
    long long fe_stride, const double* __restrict__ fi, long long fi_stride, int first,
    double phibar, const double* __restrict__ lamv, double* __restrict__ quad) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= C2) return;
  const int m = blockIdx.y;
  const double lam = lamv[e >> 1];
  const Tri a0 = load_tri(u0, C2, e);
  const Tri fi0 = f_impl_tri(a0, phibar, lam);
  Tri b = a0;
  for (int j = 0; j < M; ++j) {
    const Tri ej = load_tri(fe + j * fe_stride, C2, e);
    const Tri ij = first ? fi0 : load_tri(fi + j * fi_stride, C2, e);
    const double w = cf.v[m * M + j];
    b = axpy_tri(axpy_tri(b, w, ej), w, ij);
  }
  store_tri(quad + (size_t)m * 3 * C2, C2, e, b);
}

// node m of a serial sweep: beta = quad_m (+ corr) - alpha fi_m; u = solve;
// fi_new = f_I(u).
__global__ void __launch_bounds__(256) k_serial_node(
    int C2, double alpha, double a_phi, double a2_phi, int use_corr,
    const double* __restrict__ quad, const double* __restrict__ corr,
    const double* __restrict__ u0, const double* __restrict__ fi_old, int first, double phibar,
    const double* __restrict__ lamv, double* __restrict__ u_out, double* u_out2,
    double* __restrict__ fi_new, int* diverged, const int* step_counter,
    const double2* __restrict__ xscale, const int* __restrict__ idx_row,
    double* __restrict__ xsyn) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= C2) return;
  const double lam = lamv[e >> 1];
  Tri b = load_tri(quad, C2, e);
  if (use_corr) b = add_tri(b, load_tri(corr, C2, e));
  const Tri fo = first ? f_impl_tri(load_tri(u0, C2, e), phibar, lam) : load_tri(fi_old, C2, e);
  b = axmy_tri(b, alpha, fo);
  const Tri u = solve_tri(b, alpha, a_phi, a2_phi, lam);
  store_tri(u_out, C2, e, u);
  store_tri(fi_new, C2, e, f_impl_tri(u, phibar, lam));
  if (xsyn != nullptr)
    write_xsyn_half(xsyn + xsyn_off(idx_row[e >> 1], 0, 1), 16, e & 1, u.phi, u.zeta, u.delta,
                    xscale[e >> 1]);
  if (u_out2 != nullptr) {
    store_tri(u_out2, C2, e, u);
    if (diverged != nullptr && !finite_tri(u)) atomicMin(diverged, step_counter ? *step_counter : 1);
  }
}

// corr (+)= we (fe_new - fe_old) ; corr += wi (fi_new - fi_old)   (integrators.py:225-227)
__global__ void __launch_bounds__(256) k_serial_update(
    int C2, double we, double wi, int use_corr, double* __restrict__ corr,
    const double* __restrict__ fe_new, const double* __restrict__ fe_old,
    const double* __restrict__ fi_new, const double* __restrict__ fi_old,
    const double* __restrict__ u0, int first, double phibar, const double* __restrict__ lamv) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= C2) return;
  const double lam = lamv[e >> 1];
  const Tri en = load_tri(fe_new, C2, e), eo = load_tri(fe_old, C2, e);
  const Tri fn = load_tri(fi_new, C2, e);
  const Tri fo = first ? f_impl_tri(load_tri(u0, C2, e), phibar, lam) : load_tri(fi_old, C2, e);
  const Tri de = sub_tri(en, eo), di = sub_tri(fn, fo);
  Tri c;
  if (use_corr) {
    c = axpy_tri(load_tri(corr, C2, e), we, de);
  } else {  // the correction starts at zero: 0 + x == x
    c = Tri{__dmul_rn(we, de.phi), __dmul_rn(we, de.zeta), __dmul_rn(we, de.delta)};
  }
  store_tri(corr, C2, e, axpy_tri(c, wi, di));
}

// ---------------------------------------------------------------------------
// problem operations
// ---------------------------------------------------------------------------
__global__ void __launch_bounds__(256) k_f_impl(int C2, const double* __restrict__ u,
                                                double* __restrict__ fi, double phibar,
                                                const double* __restrict__ lamv) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= C2) return;
  const size_t b = blockIdx.y;
  store_tri(fi + b * 3 * C2, C2, e, f_impl_tri(load_tri(u + b * 3 * C2, C2, e), phibar, lamv[e >> 1]));
}

__global__ void __launch_bounds__(256) k_solve(int C2, NodeArgs cf, const double* __restrict__ beta,
                                               double* __restrict__ u,
                                               const double* __restrict__ lamv) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  const int e = blockIdx.x * blockDim.x + threadIdx.x;
  if (e >= C2) return;
  const int b = blockIdx.y;
  const Tri bt = load_tri(beta + (size_t)b * 3 * C2, C2, e);
  const double alpha = cf.v[3 * b];
  const Tri r = alpha == 0.0 ? bt : solve_tri(bt, alpha, cf.v[3 * b + 1], cf.v[3 * b + 2], lamv[e >> 1]);
  store_tri(u + (size_t)b * 3 * C2, C2, e, r);
}

// out = x + w * y element-wise, two roundings (numpy's `x + w * y`); n doubles
__global__ void __launch_bounds__(256) k_axpy(long long n, const double* __restrict__ x, double w,
                                              const double* __restrict__ y, double* out) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = __dadd_rn(x[i], __dmul_rn(w, y[i]));
}

__global__ void k_check_finite(const double* __restrict__ x, long long n, int* flag) {
  SDCSW_PDL_ENTRY();
  SDCSW_PDL_WAIT();
  long long i = blockIdx.x * (long long)blockDim.x + threadIdx.x;
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool bad = false;
  for (; i < n; i += stride) bad |= !isfinite(x[i]);
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicExch(flag, 1);
}

// ---------------------------------------------------------------------------
static inline dim3 grid_for(int C, int y = 1) { return dim3((2 * C + 255) / 256, y); }

static NodeArgs pack(const double* v, int n) {
  NodeArgs a;
  for (int k = 0; k < n && k < 16 * 20; ++k) a.v[k] = v[k];
  return a;
}

#define D(x) reinterpret_cast<const double*>(x)
#define W(x) reinterpret_cast<double*>(x)

cudaError_t launch_f_impl(const Plan& p, const double2* u, double2* fi, int nb, cudaStream_t s) {
  launch_k(k_f_impl, grid_for(p.C, nb), 256, 0, s, 2 * p.C, D(u), W(fi), p.phibar, p.lam);
  return cudaGetLastError();
}

cudaError_t launch_solve(const Plan& p, const double* coef_host, const double2* beta, double2* u,
                         int nb, cudaStream_t s) {
  // coefficients travel by value; batches above 100 states are split
  for (int b0 = 0; b0 < nb; b0 += 100) {
    const int n = nb - b0 < 100 ? nb - b0 : 100;
    launch_k(k_solve, grid_for(p.C, n), 256, 0, s, 2 * p.C, pack(coef_host + 3 * b0, 3 * n),
                                              D(beta + (size_t)b0 * 3 * p.C),
                                              W(u + (size_t)b0 * 3 * p.C), p.lam);
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) return e;
  }
  return cudaSuccess;
}

// threads per CTA of the one-thread-per-coefficient node kernels (experiment knob
// SDCSW_NODE_THREADS in {64, 128, 256}; the residual variant keeps 256)
static int node_threads() {
  static const int t = [] {
    const char* e = getenv("SDCSW_NODE_THREADS");
    const int v = e != nullptr ? atoi(e) : 256;
    return v == 64 || v == 128 || v == 256 ? v : 256;
  }();
  return t;
}

cudaError_t launch_sweep_nodes(const Plan& p, int M, int node_lo, int count, const double* coef_host,
                               const double2* u0, const double2* fe, long long fe_stride,
                               const double2* fi, long long fi_stride, int first, double2* u_out,
                               double2* fi_out, double* xsyn_out, cudaStream_t s, int members,
                               long long fe_mstride, long long fi_mstride, int chunk,
                               const PeerWait* pw, const ResidArgs* ra) {
  const long long S2 = 6LL * p.C;  // doubles per state
  const PeerWait pwv = pw != nullptr ? *pw : PeerWait{nullptr, 0, 0};
  const ResidArgs rav = ra != nullptr ? *ra : ResidArgs{nullptr, nullptr, nullptr, nullptr};
  if (ra != nullptr && (M > kFuseMaxNodes || members != 1 || p.own_idx != nullptr || count > 6))
    return cudaErrorInvalidValue;
  if (M <= kFuseMaxNodes) {  // one thread per coefficient for all nodes of the block
    dim3 grid(((p.own_idx ? p.n_own_idx : p.C) + 255) / 256, 1, members);
    if (ra != nullptr)
      launch_k(k_sweep_nodes_all<true>, grid, 256, 0, s, p.C, M, node_lo, count,
             pack(coef_host, M * (M + 4)), D(u0), D(fe), fe_stride * S2, D(fi), fi_stride * S2,
             first, p.phibar, p.lam, W(u_out), W(fi_out), p.xscale, p.idx_row, xsyn_out,
             fe_mstride * S2, fi_mstride * S2, p.rows, chunk, p.own_idx, p.n_own_idx, pwv, rav);
    else {
      const int nt = node_threads();
      grid.x = ((p.own_idx ? p.n_own_idx : p.C) + nt - 1) / nt;
      launch_k(k_sweep_nodes_all<false>, grid, nt, 0, s, p.C, M, node_lo, count,
             pack(coef_host, M * (M + 4)), D(u0), D(fe), fe_stride * S2, D(fi), fi_stride * S2,
             first, p.phibar, p.lam, W(u_out), W(fi_out), p.xscale, p.idx_row, xsyn_out,
             fe_mstride * S2, fi_mstride * S2, p.rows, chunk, p.own_idx, p.n_own_idx, pwv, rav);
    }
    return cudaGetLastError();
  }
  dim3 grid = grid_for(p.own_idx ? p.n_own_idx : p.C, count);
  grid.z = members;
  launch_k(k_sweep_nodes, grid, 256, 0, s, 2 * p.C, M, node_lo, pack(coef_host, M * (M + 4)),
                                                     D(u0), D(fe), fe_stride * S2, D(fi),
                                                     fi_stride * S2, first, p.phibar, p.lam,
                                                     W(u_out), W(fi_out), p.xscale, p.idx_row,
                                                     xsyn_out, fe_mstride * S2, fi_mstride * S2,
                                                     p.rows, chunk, p.own_idx, p.n_own_idx, pwv);
  return cudaGetLastError();
}

cudaError_t launch_sweep_nodes_po(const Plan& p, int M, int node_lo, int count, const double* coef_host,
                                  const double2* u0, const double2* fe, long long fe_stride,
                                  const double2* fi, long long fi_stride, int first, double2* fi_out,
                                  double* xsp, cudaStream_t s, int members, long long fe_mstride,
                                  long long fi_mstride) {
  if (M > kFuseMaxNodes || p.coef_prow == nullptr || xsp == nullptr || p.own_idx != nullptr)
    return cudaErrorInvalidValue;
  const long long S2 = 6LL * p.C;
  const int warps = (p.C + 29) / 30;  // 30 coefficients per warp (+ 2 halo lanes)
  dim3 grid((warps + 7) / 8, 1, members);
  launch_k(k_sweep_nodes_po, grid, 256, 0, s, p.C, M, node_lo, count, pack(coef_host, M * (M + 4)),
           D(u0), D(fe), fe_stride * S2, D(fi), fi_stride * S2, first, p.phibar, p.lam, W(fi_out),
           p.xscale, p.coef_prow, p.cvt_ab, xsp, fe_mstride * S2, fi_mstride * S2);
  return cudaGetLastError();
}

cudaError_t launch_final_node(const Plan& p, int M, const double* coef_host, const double2* u0,
                              const double2* fe, long long fe_stride, const double2* fi,
                              long long fi_stride, int first, double2* u_out, int* diverged,
                              const int* step_counter, double* xsyn_out, cudaStream_t s,
                              int members, long long fe_mstride, long long fi_mstride,
                              const PeerWait* pw) {
  const long long S2 = 6LL * p.C;
  const PeerWait pwv = pw != nullptr ? *pw : PeerWait{nullptr, 0, 0};
  const int nt = node_threads();
  dim3 grid(((p.own_idx ? p.n_own_idx : p.C) + nt - 1) / nt, 1, members);
  launch_k(k_final_node_c, grid, nt, 0, s, p.C, M, pack(coef_host, M + 4), D(u0), D(fe),
                                             fe_stride * S2, D(fi), fi_stride * S2, first, p.phibar,
                                             p.lam, W(u_out), diverged, step_counter, p.xscale,
                                             p.idx_row, xsyn_out, fe_mstride * S2, fi_mstride * S2,
                                             p.rows, p.fe_chunk, p.own_idx, p.n_own_idx, pwv);
  return cudaGetLastError();
}

cudaError_t launch_serial_quad(const Plan& p, int M, const double* w_host, const double2* u0,
                               const double2* fe, long long fe_stride, const double2* fi,
                               long long fi_stride, int first, double2* quad, cudaStream_t s) {
  const long long S2 = 6LL * p.C;
  launch_k(k_serial_quad, grid_for(p.C, M), 256, 0, s, 2 * p.C, M, pack(w_host, M * M), D(u0), D(fe),
                                                 fe_stride * S2, D(fi), fi_stride * S2, first,
                                                 p.phibar, p.lam, W(quad));
  return cudaGetLastError();
}

cudaError_t launch_serial_node(const Plan& p, int M, int m, const double* coef_host,
                               const double2* quad, const double2* corr, const double2* u0,
                               const double2* fi_old, int first, double2* u_out, double2* u_out2,
                               double2* fi_new, int* diverged, const int* step_counter,
                               double* xsyn_out, cudaStream_t s) {
  (void)M;
  launch_k(k_serial_node, grid_for(p.C), 256, 0, s, 2 * p.C, coef_host[0], coef_host[1], coef_host[2],
                                              m > 0, D(quad), D(corr), D(u0), D(fi_old), first,
                                              p.phibar, p.lam, W(u_out), W(u_out2), W(fi_new),
                                              diverged, step_counter, p.xscale, p.idx_row,
                                              xsyn_out);
  return cudaGetLastError();
}

cudaError_t launch_serial_update(const Plan& p, int m, double we, double wi, double2* corr,
                                 const double2* fe_new, const double2* fe_old,
                                 const double2* fi_new, const double2* fi_old, const double2* u0,
                                 int first, cudaStream_t s) {
  launch_k(k_serial_update, grid_for(p.C), 256, 0, s, 2 * p.C, we, wi, m > 0, W(corr), D(fe_new),
                                                D(fe_old), D(fi_new), D(fi_old), D(u0), first,
                                                p.phibar, p.lam);
  return cudaGetLastError();
}

cudaError_t launch_axpy(long long n, const double* x, double w, const double* y, double* out,
                        cudaStream_t s) {
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 16) blocks = 148 * 16;
  if (blocks < 1) blocks = 1;
  launch_k(k_axpy, dim3((unsigned)blocks), 256, 0, s, n, x, w, y, out);
  return cudaGetLastError();
}

cudaError_t launch_check_finite(const double* x, long long n, int* flag, cudaStream_t s) {
  long long blocks = (n + 255) / 256;
  if (blocks > 148 * 8) blocks = 148 * 8;
  if (blocks < 1) blocks = 1;
  launch_k(k_check_finite, (unsigned)blocks, 256, 0, s, x, n, flag);
  return cudaGetLastError();
}

}  // namespace sdcsw
