// Table-streaming Legendre analysis for large truncations (T >= 400, where the
// P/H tables - 403 MB each at T511 - live in HBM, not L2).
//
// The A operand (table rows x latitudes) is streamed into shared memory by the
// Tensor Memory Accelerator: cp.async.bulk.tensor.2d boxes of 64 rows x 16
// latitudes (8 KB per table), 128-byte swizzled, completing on an mbarrier,
// in a kStages-deep ring.  One elected thread issues the copies; the four
// warps (one 16-row tile each) read DMMA A fragments from the swizzled tiles
// and B fragments (analysis data, shared by all four warps) through L1.  The
// table stream is thus decoupled from register prefetching, which is what
// limited the register-only kernel (k_analysis) at T511.
//
// Same contraction and epilogue as k_analysis in legendre.cu:
//   out[n,c] = sum_j P[n,j] Xfold[j,c] + sum_j H[n,j] Yfold[j,c]
//   (pkg/src/parsdc/problems/swe.py:180-190 restated on the sphere).
#include <cstdlib>
#include <cuda.h>
#include <cudaTypedefs.h>

#include "internal.cuh"

namespace sdcsw {

constexpr int kTmaRows = 64;   // table rows per CTA (4 warps x 16)
constexpr int kTmaLat = 16;    // latitudes per stage (128 B per row, the swizzle span)
constexpr int kStages = 4;
constexpr int kTileBytes = kTmaRows * kTmaLat * 8;  // 8 KB per table per stage

__device__ __forceinline__ void dmma_t(double (&c)[2], double a, double b) {
  asm("mma.sync.aligned.m8n8k4.row.col.f64.f64.f64.f64 {%0,%1}, {%2}, {%3}, {%0,%1};"
      : "+d"(c[0]), "+d"(c[1])
      : "d"(a), "d"(b));
}

__device__ __forceinline__ void tma_load_2d(void* dst, const CUtensorMap* map, int x, int y,
                                            unsigned long long* bar) {
  asm volatile(
      "cp.async.bulk.tensor.2d.shared::cluster.global.tile.mbarrier::complete_tx::bytes"
      " [%0], [%1, {%2, %3}], [%4];" ::"r"(smem_u32(dst)),
      "l"(reinterpret_cast<unsigned long long>(map)), "r"(x), "r"(y), "r"(smem_u32(bar))
      : "memory");
}

// element (row, k) of a 128B-swizzled [rows][16] double tile
__device__ __forceinline__ double swz(const double* tile, int row, int k) {
  const int chunk = (k >> 1) ^ (row & 7);
  return tile[row * 16 + chunk * 2 + (k & 1)];
}

template <int NB>
__global__ void __launch_bounds__(128) k_analysis_tma(
    const __grid_constant__ CUtensorMap pmap, const __grid_constant__ CUtensorMap hmap,
    const double2* __restrict__ gan, int nb, int T, int J, int C, const int* __restrict__ rowoff,
    const int* __restrict__ n_even, const int* __restrict__ row_n, const int* __restrict__ moff,
    const double* __restrict__ lam, const int* __restrict__ work, double2* __restrict__ fe) {
  SDCSW_PDL_ENTRY();
  constexpr int PC = 8 * NB;
  constexpr int OS = PC + 1;
  extern __shared__ __align__(1024) unsigned char tma_smem[];
  double* ptile = reinterpret_cast<double*>(tma_smem);                    // [kStages][64][16]
  double* htile = reinterpret_cast<double*>(tma_smem + kStages * kTileBytes);
  unsigned long long* full =
      reinterpret_cast<unsigned long long*>(tma_smem + 2 * kStages * kTileBytes);

  const int wk = work[blockIdx.x];
  const int m = wk >> 16, rb = wk & 0xffff;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int b0 = blockIdx.y * NB;
  const int L = T + 1;
  const int r0m = rowoff[m];
  const int rows = rowoff[m + 1] - r0m;
  const int le = n_even[m];
  const int rblock = r0m + rb * kTmaRows;  // first table row of this CTA
  const int rw = rb * kTmaRows + warp * kRowsPerWarp;
  const bool live = rw < rows;
  const bool ev0 = rw < le, ev1 = rw + 8 < le;
  const int nchunks = J / kTmaLat;

  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  // the tables are constant: start streaming before waiting for the producer kernel
  if (threadIdx.x == 0) {
    for (int s = 0; s < kStages && s < nchunks; ++s) {
      mbar_expect_tx(&full[s], 2 * kTileBytes);
      tma_load_2d(ptile + s * kTmaRows * kTmaLat, &pmap, s * kTmaLat, rblock, &full[s]);
      tma_load_2d(htile + s * kTmaRows * kTmaLat, &hmap, s * kTmaLat, rblock, &full[s]);
    }
  }
  SDCSW_PDL_WAIT();

  // B column tiles: tile c = state b0 + c.  P columns g = 2 slot + re/im over
  // (X_phi, X_zeta, X_delta, X_ke); H columns g < 6 over (Y_phi, Y_zeta,
  // Y_delta), accumulated into the same outputs.  Fragment-order analysis data
  // (gan_off): the lanes of one tile read 32 (P) or 24 (H) consecutive doubles.
  const double* gb = reinterpret_cast<const double*>(gan);
  long long bbase[NB];
#pragma unroll
  for (int c = 0; c < NB; ++c)
    bbase[c] = b0 + c < nb ? ((long long)(b0 + c) * L + m) * J * 28 + t * 8 + g : -1;
  const int hsh = 32 + t * 6 + g - (t * 8 + g);
  const bool hcol = g < 6;
  const bool any_ev = ev0 || ev1, any_od = !ev0 || !ev1;

  double acc[2][NB][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < NB; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;

  const int row0 = warp * kRowsPerWarp + g;  // tile rows of this lane (a = 0; a = 1 adds 8)
  struct BFrag {
    double ps[NB], pa[NB], hs[NB], ha[NB];
  };
  auto fetch_b = [&](int lat, BFrag& f) {  // lat = 4 s + t
    const long long ks112 = (long long)(lat >> 2) * 112;
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      const bool ok = bbase[c] >= 0;
      const double* q = gb + bbase[c] + ks112;
      f.ps[c] = ok && any_ev ? __ldg(q) : 0.0;
      f.pa[c] = ok && any_od ? __ldg(q + 56) : 0.0;
      f.hs[c] = ok && any_od && hcol ? __ldg(q + hsh) : 0.0;
      f.ha[c] = ok && any_ev && hcol ? __ldg(q + 56 + hsh) : 0.0;
    }
  };
  BFrag cur, nxt;
  fetch_b(t, cur);  // latitude 4 q + t of chunk 0, q = 0
  for (int ch = 0; ch < nchunks; ++ch) {
    const int st = ch % kStages;
    mbar_wait(&full[st], (ch / kStages) & 1);
    const double* pt = ptile + st * kTmaRows * kTmaLat;
    const double* ht = htile + st * kTmaRows * kTmaLat;
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      // B of the next k-step (next chunk's first after q = 3), loaded ahead
      const int nl = q < 3 ? ch * kTmaLat + 4 * (q + 1) + t
                           : (ch + 1 < nchunks ? (ch + 1) * kTmaLat + t : ch * kTmaLat + t);
      fetch_b(nl, nxt);
      if (live) {
        const int k = 4 * q + t;
        const double aP0 = swz(pt, row0, k), aP1 = swz(pt, row0 + 8, k);
        const double aH0 = swz(ht, row0, k), aH1 = swz(ht, row0 + 8, k);
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          dmma_t(acc[0][c], aP0, ev0 ? cur.ps[c] : cur.pa[c]);
          dmma_t(acc[1][c], aP1, ev1 ? cur.ps[c] : cur.pa[c]);
        }
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          dmma_t(acc[0][c], aH0, ev0 ? cur.ha[c] : cur.hs[c]);
          dmma_t(acc[1][c], aH1, ev1 ? cur.ha[c] : cur.hs[c]);
        }
      }
      cur = nxt;
    }
    __syncthreads();  // every warp is done with stage st
    if (threadIdx.x == 0 && ch + kStages < nchunks) {
      const int nc = ch + kStages;
      mbar_expect_tx(&full[st], 2 * kTileBytes);
      tma_load_2d(ptile + st * kTmaRows * kTmaLat, &pmap, nc * kTmaLat, rblock, &full[st]);
      tma_load_2d(htile + st * kTmaRows * kTmaLat, &hmap, nc * kTmaLat, rblock, &full[st]);
    }
  }
  if (!live) return;
  // epilogue through a per-warp shared tile (reuses the stage buffers: all
  // copies completed and were consumed before the last barrier)
  double* o = ptile + warp * kRowsPerWarp * OS;
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      o[(8 * a + g) * OS + 8 * c + 2 * t] = acc[a][c][0];
      o[(8 * a + g) * OS + 8 * c + 2 * t + 1] = acc[a][c][1];
    }
  __syncwarp();
  const int mo = moff[m];
  for (int it = lane; it < kRowsPerWarp * NB; it += 32) {
    const int rr = it % kRowsPerWarp, b = it / kRowsPerWarp;
    if (rw + rr >= rows || b0 + b >= nb) continue;
    const int n = row_n[r0m + rw + rr];
    if (n < 0) continue;
    const int idx = mo + n - m;
    const double* row = o + rr * OS;
    const double l = lam[idx];
    double2 phi = make_double2(row[8 * b + 0], row[8 * b + 1]);
    double2 zeta = make_double2(row[8 * b + 2], row[8 * b + 3]);
    double2 delta = make_double2(__fma_rn(l, row[8 * b + 6], row[8 * b + 4]),
                                 __fma_rn(l, row[8 * b + 7], row[8 * b + 5]));
    if (m == 0) phi.y = zeta.y = delta.y = 0.0;
    double2* dst = fe + (size_t)(b0 + b) * 3 * C;
    dst[idx] = phi;
    dst[C + idx] = zeta;
    dst[2 * C + idx] = delta;
  }
}

constexpr size_t kTmaSmem = 2 * kStages * kTileBytes + 64;

static_assert(kRowsPerWarp * (8 * 6 + 1) * 4 * 8 <= 2 * kStages * kTileBytes,
              "epilogue tiles fit in the stage buffers");

// Tensor maps over the packed tables: dims {J, rows + 16}, box {16, 64},
// 128-byte swizzle; out-of-range rows read as zero.
cudaError_t make_table_maps(Plan& p) {
  p.tma_ok = false;
  const char* env = getenv("SDCSW_TMA_MIN_T");  // table-streaming analysis from this truncation
  // from T200: with the B operand staged (k_analysis_bulk) the unfused step beats the
  // fused latency-regime analysis at T255 (c2 1985 vs 1866 steps/s); not at T127/T63
  // for one state, but for ensemble plans (p.ensemble) at every truncation
  const int tmin = env ? atoi(env) : (p.ensemble ? 0 : 200);
  if (p.T < tmin || p.J % kTmaLat) return cudaSuccess;
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || !fn || q != cudaDriverEntryPointSuccess) return cudaSuccess;
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  const cuuint64_t dims[2] = {(cuuint64_t)p.J, (cuuint64_t)p.rows + 16};
  const cuuint64_t strides[1] = {(cuuint64_t)p.J * sizeof(double)};
  const cuuint32_t box[2] = {kTmaLat, kTmaRows};
  const cuuint32_t elem[2] = {1, 1};
  double* tabs[2] = {p.ptab, p.htab};
  for (int i = 0; i < 2; ++i) {
    CUresult r = encode(reinterpret_cast<CUtensorMap*>(&p.tmap[i]), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                        tabs[i], dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                        CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                        CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
    if (r != CUDA_SUCCESS) return cudaSuccess;  // fall back to k_analysis (also sm_100a)
  }
#define SDCSW_TMA_ATTR(NBV)                                                                     \
  e = cudaFuncSetAttribute(k_analysis_tma<NBV>, cudaFuncAttributeMaxDynamicSharedMemorySize,    \
                           (int)kTmaSmem);                                                      \
  if (e != cudaSuccess) return e;
  SDCSW_TMA_ATTR(1) SDCSW_TMA_ATTR(2) SDCSW_TMA_ATTR(3) SDCSW_TMA_ATTR(4) SDCSW_TMA_ATTR(5)
  SDCSW_TMA_ATTR(6)
#undef SDCSW_TMA_ATTR
  p.tma_ok = true;
  return cudaSuccess;
}

static cudaError_t launch_analysis_bulk(const Plan& p, const Work& w, double2* fe, int nb,
                                        int NB, const int* work, int nwork, cudaStream_t s);

bool launch_analysis_tma(const Plan& p, const Work& w, double2* fe, int nb, cudaStream_t s,
                         cudaError_t* err) {
  if (!tma_active(p)) return false;
  int NB = nb <= 6 ? nb : 4;
  if (p.ana_nb > 0 && NB > p.ana_nb) NB = p.ana_nb;  // states per CTA (columns per B tile)
  const int* work = p.own_work != nullptr ? p.own_work : p.anal_work;
  const int nwork = p.own_work != nullptr ? p.n_own_work : p.n_anal_work;
  if (p.ana_bulk != 0) {  // B operand staged with the tables (default)
    *err = launch_analysis_bulk(p, w, fe, nb, NB, work, nwork, s);
    return true;
  }
  dim3 grid(nwork, (nb + NB - 1) / NB);
  const CUtensorMap& pm = *reinterpret_cast<const CUtensorMap*>(&p.tmap[0]);
  const CUtensorMap& hm = *reinterpret_cast<const CUtensorMap*>(&p.tmap[1]);
#define SDCSW_TMA_LAUNCH(NBV)                                                                  \
  if (NB == NBV) {                                                                             \
    *err = launch_k(k_analysis_tma<NBV>, grid, dim3(128), kTmaSmem, s, pm, hm, w.gan, nb, p.T,  \
                    p.J, p.C, p.rowoff, p.n_even, p.row_n, p.moff, p.lam, work, fe);           \
    return true;                                                                               \
  }
  SDCSW_TMA_LAUNCH(1) SDCSW_TMA_LAUNCH(2) SDCSW_TMA_LAUNCH(3) SDCSW_TMA_LAUNCH(4)
  SDCSW_TMA_LAUNCH(5) SDCSW_TMA_LAUNCH(6)
#undef SDCSW_TMA_LAUNCH
  return false;
}

// ---------------------------------------------------------------------------
// Table-streaming Legendre synthesis (large truncations): CTA-staged operands.
//
// k_synthesis_cp stages every warp's own A and B fragments with 16-byte
// cp.async copies; at T511 that costs ~280 instructions (address arithmetic,
// copies, waits) per 18 DMMAs, so the kernel is issue-bound with the DMMA pipe
// ~57% busy.  Here one thread feeds a kSynBS-deep ring of stages with bulk
// copies (cp.async.bulk, completing on an mbarrier): per stage kSynKQ row
// quads of the CTA's P and H slices (WJ x 2 latitude octets, contiguous in the
// fragment-ordered tables) and the operand records of the same rows for all
// states (contiguous too: [row/4][part][state][row%4][4]).  The operand is
// staged once per CTA instead of once per warp, and the K loop is LDS + DMMA
// only.  Same contraction, parity handling and output as k_synthesis_cp, with
// no K-split (the sums run over k in the same order as its WK = 1 plan).
// ---------------------------------------------------------------------------
#ifndef SDCSW_SYNB_STAGES
#define SDCSW_SYNB_STAGES 2
#endif
#ifndef SDCSW_SYNB_KQ
#define SDCSW_SYNB_KQ 4
#endif
#ifndef SDCSW_SYNB_MINB
#define SDCSW_SYNB_MINB 4  // resident CTAs per SM (NB > 2): 16 warps, <= 128 registers
#endif
#ifndef SDCSW_SYNB_MINB1
#define SDCSW_SYNB_MINB1 6  // NB <= 2
#endif
constexpr int kSynKQ = SDCSW_SYNB_KQ;      // row quads (4 table rows each) per stage
constexpr int kSynBS = SDCSW_SYNB_STAGES;  // stages in flight

// PO (H-free path, legendre_ponly.cu): one table (P to degree T+1) and two operand parts
// kq: row quads per stage (the H-free kernel takes 8 from T400: T511 5 states 180 -> 168 us;
// 4 elsewhere, where 8 measured slower)
__host__ __device__ constexpr int synb_stage_doubles(int wj, int nbt, bool po = false, int kq = kSynKQ) {
  return po ? kq * (wj * 64 + 32 * nbt) + 16
            : kq * (2 * wj * 64 + 48 * nbt) + 16;  // + pad: odd-pair reads past the last quad
}
__host__ __device__ constexpr size_t synb_smem(int wj, int nbt, bool po = false, int kq = kSynKQ) {
  return (size_t)kSynBS * synb_stage_doubles(wj, nbt, po, kq) * 8 + 8 * kSynBS;
}


template <int NB, bool PO, int KQ = kSynKQ>
__global__ void __launch_bounds__(128, NB <= 2 ? SDCSW_SYNB_MINB1 : SDCSW_SYNB_MINB) k_synthesis_bulk(
    const double* __restrict__ xsyn, int nb, int J, const double* __restrict__ ptab,
    const double* __restrict__ htab, const int* __restrict__ rowoff,
    const int* __restrict__ n_even, double2* __restrict__ fsyn, int* step_counter,
    const int* __restrict__ mlist, int Lp, const SynDst sd) {
  SDCSW_PDL_ENTRY();
  // column tiles: NB / 2 state pairs x (part 0, part 1) for P plus one H tile per
  // pair; an odd last state gets one P tile holding both its parts (columns 0-3
  // part 0, 4-7 part 1) and one H tile (columns 0-3, the rest zero) accumulating
  // into it, instead of a pair tile with an empty partner (NB = 5: 16 DMMAs per row
  // quad instead of 18; per-column sums unchanged)
  constexpr int NFULL = NB / 2;
  constexpr bool ODD = (NB & 1) != 0;
  constexpr int NT = 2 * NFULL + (ODD ? 1 : 0);  // P tiles
  constexpr int NH = NFULL + (ODD ? 1 : 0);      // H tiles (none when PO)
  constexpr int NPART = PO ? 2 : 3;              // operand parts
  constexpr int NTAB = PO ? 1 : 2;               // tables streamed
  constexpr int QX = 16 * NPART * NB;  // operand doubles per row quad (parts x NB states x 16)
  extern __shared__ __align__(128) unsigned char synb_raw[];
  const int WJ = blockDim.x >> 5;
  const int SD = synb_stage_doubles(WJ, NB, PO, KQ);
  const int TQ = WJ * 64;  // table doubles per row quad of this CTA's latitudes
  double* stages = reinterpret_cast<double*>(synb_raw);
  unsigned long long* full = reinterpret_cast<unsigned long long*>(synb_raw + (size_t)kSynBS * SD * 8);

  const int kpos = blockIdx.y;
  const int m = mlist != nullptr ? mlist[kpos] : kpos;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int gb = g >> 2, gc = g & 3;
  const int j0 = (blockIdx.x * WJ + warp) * kRowsPerWarp;
  const int r0m = rowoff[m];
  const int nsteps = (rowoff[m + 1] - r0m) >> 2;
  const int se = n_even[m] >> 2;
  const int nstage = (nsteps + KQ - 1) / KQ;
  const size_t qstride = (size_t)(J / 8) * 32;
  const double* Pc = ptab + (size_t)(r0m / 4) * qstride + (size_t)blockIdx.x * TQ;
  const double* Hc = htab + (size_t)(r0m / 4) * qstride + (size_t)blockIdx.x * TQ;
  // batch block blockIdx.z: states [b0, b0 + nbv) of nb; operand records are
  // [row/4][part][nb][16], one contiguous run per quad when the block is the batch
  const int b0 = blockIdx.z * NB, nbv = nb - b0 < NB ? nb - b0 : NB;
  const size_t qxg = (size_t)16 * NPART * nb;  // operand doubles per row quad (all states)
  const double* Xc = xsyn + (size_t)(r0m / 4) * qxg + (size_t)b0 * 16;

  auto nq_of = [&](int i) { return min(KQ, nsteps - i * KQ); };
  auto issue_tables = [&](int i) {  // thread 0
    double* st = stages + (i % kSynBS) * SD;
    const int nq = nq_of(i);
    mbar_expect_tx(&full[i % kSynBS], (unsigned)(nq * (NTAB * TQ + 16 * NPART * nbv) * 8));
    for (int q = 0; q < nq; ++q) {
      const size_t src = (size_t)(i * KQ + q) * qstride;
      bulk_g2s(st + q * TQ, Pc + src, TQ * 8, &full[i % kSynBS]);
      if constexpr (!PO) bulk_g2s(st + (KQ + q) * TQ, Hc + src, TQ * 8, &full[i % kSynBS]);
    }
  };
  auto issue_operand = [&](int i) {  // thread 0, after the producer grid completed
    double* st = stages + (i % kSynBS) * SD + NTAB * KQ * TQ;
    if (nb == NB) {
      bulk_g2s(st, Xc + (size_t)i * KQ * QX, (unsigned)(nq_of(i) * QX * 8), &full[i % kSynBS]);
    } else {  // one run of nbv states per (quad, part), placed at the block's [part][NB] stride
      for (int q = 0; q < nq_of(i); ++q)
        for (int pp = 0; pp < NPART; ++pp)
          bulk_g2s(st + q * QX + pp * 16 * NB, Xc + (size_t)(i * KQ + q) * qxg + pp * 16 * nb,
                   (unsigned)(nbv * 16 * 8), &full[i % kSynBS]);
    }
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kSynBS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  // the tables are constant: start streaming them before the producer grid ends
  if (threadIdx.x == 0)
    for (int i = 0; i < kSynBS && i < nstage; ++i) issue_tables(i);
  SDCSW_PDL_WAIT();
  if (threadIdx.x == 0) {
    if (step_counter != nullptr && (blockIdx.x | blockIdx.y | blockIdx.z) == 0) atomicAdd(step_counter, 1);
    for (int i = 0; i < kSynBS && i < nstage; ++i) issue_operand(i);
  }

  double aE[2][NT][2], aO[2][NT][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < NT; ++c) aE[a][c][0] = aE[a][c][1] = aO[a][c][0] = aO[a][c][1] = 0.0;

  for (int i = 0; i < nstage; ++i) {
    mbar_wait(&full[i % kSynBS], (i / kSynBS) & 1);
    const double* st = stages + (i % kSynBS) * SD;
    const int nq = nq_of(i);
#pragma unroll
    for (int q = 0; q < KQ; ++q) {
      if (q < nq) {
        const double* pq = st + q * TQ + warp * 64 + lane;
        const double* hq = pq + KQ * TQ;
        const double aP0 = pq[0], aP1 = pq[32];
        const double aH0 = PO ? 0.0 : hq[0], aH1 = PO ? 0.0 : hq[32];
        const double* xq0 = st + NTAB * KQ * TQ + q * QX + t * 4 + gc;
        const double* xq = xq0 + gb * 16;
        double bP[NT], bH[NH];
#pragma unroll
        for (int p = 0; p < NFULL; ++p) {
          bP[2 * p] = xq[p * 32];
          bP[2 * p + 1] = xq[16 * NB + p * 32];
          bH[p] = PO ? 0.0 : xq[32 * NB + p * 32];
        }
        if constexpr (ODD) {  // last state: lane column group gb = part
          bP[NT - 1] = xq0[gb * 16 * NB + (NB - 1) * 16];
          bH[NH - 1] = !PO && gb == 0 ? xq0[32 * NB + (NB - 1) * 16] : 0.0;
        }
        if constexpr (PO) {  // H-free: every operand column is a P column
          if (i * KQ + q < se) {
#pragma unroll
            for (int c = 0; c < NT; ++c) { dmma_t(aE[0][c], aP0, bP[c]); dmma_t(aE[1][c], aP1, bP[c]); }
          } else {
#pragma unroll
            for (int c = 0; c < NT; ++c) { dmma_t(aO[0][c], aP0, bP[c]); dmma_t(aO[1][c], aP1, bP[c]); }
          }
        } else if (i * KQ + q < se) {  // n - m even: P symmetric (E), H antisymmetric (O)
#pragma unroll
          for (int c = 0; c < NT; ++c) { dmma_t(aE[0][c], aP0, bP[c]); dmma_t(aE[1][c], aP1, bP[c]); }
#pragma unroll
          for (int p = 0; p < NH; ++p) {
            const int c = p < NFULL ? 2 * p : NT - 1;
            dmma_t(aO[0][c], aH0, bH[p]); dmma_t(aO[1][c], aH1, bH[p]);
          }
        } else {
#pragma unroll
          for (int c = 0; c < NT; ++c) { dmma_t(aO[0][c], aP0, bP[c]); dmma_t(aO[1][c], aP1, bP[c]); }
#pragma unroll
          for (int p = 0; p < NH; ++p) {
            const int c = p < NFULL ? 2 * p : NT - 1;
            dmma_t(aE[0][c], aH0, bH[p]); dmma_t(aE[1][c], aH1, bH[p]);
          }
        }
      }
    }
    __syncthreads();  // every warp is done with this stage
    if (threadIdx.x == 0 && i + kSynBS < nstage) {
      issue_tables(i + kSynBS);
      issue_operand(i + kSynBS);
    }
  }

#pragma unroll
  for (int c = 0; c < NT; ++c) {
    const bool last = ODD && c == NT - 1;  // the odd state's tile: column pair t = field t
    const int be = last ? NB - 1 : 2 * (c >> 1) + (t >> 1);
    const int f = last ? t : (t & 1) + 2 * (c & 1);
    // the last batch block may hold nbv < NB states: columns of the missing states
    // were formed from stale stage memory and must not be stored
    if (be >= nbv) continue;
#pragma unroll
    for (int a = 0; a < 2; ++a) {
      const int j = j0 + 8 * a + g;
      const size_t off = ((((size_t)(b0 + be) * J + j) * Lp + kpos) * 4 + f) * 2;
      const double2 vn = make_double2(aE[a][c][0] + aO[a][c][0], aE[a][c][1] + aO[a][c][1]);
      const double2 vs = make_double2(aE[a][c][0] - aO[a][c][0], aE[a][c][1] - aO[a][c][1]);
      if (sd.n == 0) {
        fsyn[off] = vn;
        fsyn[off + 1] = vs;
      } else {  // spectral split over peer memory: every spectral peer's buffer
        const long long par = (long long)((*sd.fseq + 1) & 1) * sd.par_stride;
        for (int q = 0; q < sd.n; ++q) {
          sd.dst[q][par + off] = vn;
          sd.dst[q][par + off + 1] = vs;
        }
      }
    }
  }
}

cudaError_t configure_synthesis_bulk() {
  cudaError_t e = cudaSuccess;
#define SDCSW_SYNB_CFG(NBV)                                                                   \
  if (e == cudaSuccess)                                                                       \
    e = cudaFuncSetAttribute(k_synthesis_bulk<NBV, false>,                                    \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)synb_smem(4, NBV)); \
  if (e == cudaSuccess)                                                                       \
    e = cudaFuncSetAttribute(k_synthesis_bulk<NBV, true>,                                     \
                             cudaFuncAttributeMaxDynamicSharedMemorySize,                     \
                             (int)synb_smem(4, NBV, true));                                   \
  if (e == cudaSuccess)                                                                       \
    e = cudaFuncSetAttribute(k_synthesis_bulk<NBV, true, 8>,                                  \
                             cudaFuncAttributeMaxDynamicSharedMemorySize,                     \
                             (int)synb_smem(4, NBV, true, 8));
  SDCSW_SYNB_CFG(1) SDCSW_SYNB_CFG(2) SDCSW_SYNB_CFG(3) SDCSW_SYNB_CFG(4) SDCSW_SYNB_CFG(5)
  SDCSW_SYNB_CFG(6)
#undef SDCSW_SYNB_CFG
  return e;
}

// any nb: batch blocks of up to 6 states along grid z (the last block may be partial;
// its missing columns are not stored)
bool synthesis_bulk_ok(const Plan& p, int nb) {
  // automatic from T200 (T255 4 states 32.5 vs 38.6 us; one state 24 vs 30 us), and for
  // ensemble batches (4+ batch blocks of 6 states) at any truncation
  const int on = p.syn_bulk >= 0 ? p.syn_bulk : (p.T >= 200 || nb >= 24 ? 1 : 0);
  return on && nb >= 1 && p.J % 32 == 0;
}

cudaError_t launch_synthesis_bulk(const Plan& p, double2* fsyn, const int* mlist, int nm, int Lp,
                                  const double* xsyn, int nb, cudaStream_t s, int* step_counter,
                                  const SynDst& sd) {
  const int WJ = p.J % 64 == 0 ? 4 : 2;
  const int NB = nb <= 6 ? nb : 6;  // states per CTA (batch blocks along z)
  const dim3 grid(p.J / (kRowsPerWarp * WJ), nm, (nb + NB - 1) / NB);
#define SDCSW_SYNB_LAUNCH(NBV)                                                                \
  if (NB == NBV)                                                                              \
    return launch_k(k_synthesis_bulk<NBV, false>, grid, dim3(32 * WJ), synb_smem(WJ, NBV), s,  \
                    xsyn, nb, p.J, p.ptab_s, p.htab_s, p.rowoff, p.n_even, fsyn, step_counter,  \
                    mlist, Lp, sd);
  SDCSW_SYNB_LAUNCH(1) SDCSW_SYNB_LAUNCH(2) SDCSW_SYNB_LAUNCH(3) SDCSW_SYNB_LAUNCH(4)
  SDCSW_SYNB_LAUNCH(5) SDCSW_SYNB_LAUNCH(6)
#undef SDCSW_SYNB_LAUNCH
  return cudaErrorInvalidValue;
}

// H-free synthesis (legendre_ponly.cu): xsp = the P-only operand of the chain, P rows to T+1
cudaError_t launch_synthesis_bulk_ponly(const Plan& p, double2* fsyn, const int* mlist, int nm,
                                        int Lp, const double* xsp, int nb, cudaStream_t s,
                                        int* step_counter, const SynDst& sd) {
  const int WJ = p.J % 64 == 0 ? 4 : 2;
  const int NB = nb <= 6 ? nb : 6;
  const dim3 grid(p.J / (kRowsPerWarp * WJ), nm, (nb + NB - 1) / NB);
#define SDCSW_SYNP_LAUNCH(NBV)                                                                 \
  if (NB == NBV) {                                                                             \
    if (p.T >= 400)                                                                            \
      return launch_k(k_synthesis_bulk<NBV, true, 8>, grid, dim3(32 * WJ),                     \
                      synb_smem(WJ, NBV, true, 8), s, xsp, nb, p.J, p.ptabP_s, p.ptabP_s,     \
                      p.rowoffP, p.n_evenP, fsyn, step_counter, mlist, Lp, sd);              \
    return launch_k(k_synthesis_bulk<NBV, true>, grid, dim3(32 * WJ), synb_smem(WJ, NBV, true), \
                    s, xsp, nb, p.J, p.ptabP_s, p.ptabP_s, p.rowoffP, p.n_evenP, fsyn,          \
                    step_counter, mlist, Lp, sd);                                               \
  }
  SDCSW_SYNP_LAUNCH(1) SDCSW_SYNP_LAUNCH(2) SDCSW_SYNP_LAUNCH(3) SDCSW_SYNP_LAUNCH(4)
  SDCSW_SYNP_LAUNCH(5) SDCSW_SYNP_LAUNCH(6)
#undef SDCSW_SYNP_LAUNCH
  return cudaErrorInvalidValue;
}

// ---------------------------------------------------------------------------
// Table-streaming analysis with the B operand staged too (k_analysis_bulk).
//
// k_analysis_tma streams the tables by TMA but loads the analysis-data B
// fragments per lane from global memory, prefetched one k-step ahead in
// registers (~80 of its 168), which costs residency and ~200 instructions per
// 20 DMMAs.  Here each stage also carries, per state, the 16 latitudes x 28
// doubles of analysis data the chunk needs (one contiguous 3.5 KB bulk copy in
// the fragment order the ring kernel writes), completing on the same mbarrier
// as the table tiles; the K loop reads A and B from shared memory only.  Same
// sums in the same order as k_analysis_tma (bitwise equal), same epilogue.
// ---------------------------------------------------------------------------
#ifndef SDCSW_ANAB_STAGES
#define SDCSW_ANAB_STAGES 2
#endif
#ifndef SDCSW_ANAB_MINB
#define SDCSW_ANAB_MINB 3
#endif
constexpr int kAnbS = SDCSW_ANAB_STAGES;
constexpr int kAnbChunk = kTmaLat * 28;  // analysis-data doubles per state per stage
template <int NB>
constexpr size_t anab_smem() {
  return (size_t)kAnbS * (2 * kTileBytes + NB * kAnbChunk * 8) + 8 * kAnbS;
}

template <int NB>
__global__ void __launch_bounds__(128, SDCSW_ANAB_MINB) k_analysis_bulk(
    const __grid_constant__ CUtensorMap pmap, const __grid_constant__ CUtensorMap hmap,
    const double2* __restrict__ gan, int nb, int T, int J, int C, const int* __restrict__ rowoff,
    const int* __restrict__ n_even, const int* __restrict__ row_n, const int* __restrict__ moff,
    const double* __restrict__ lam, const int* __restrict__ work, double2* __restrict__ fe) {
  SDCSW_PDL_ENTRY();
  constexpr int PC = 8 * NB;
  constexpr int OS = PC + 1;
  extern __shared__ __align__(1024) unsigned char anb_smem[];
  double* ptile = reinterpret_cast<double*>(anb_smem);  // [kAnbS][64][16], swizzled
  double* htile = reinterpret_cast<double*>(anb_smem + kAnbS * kTileBytes);
  double* btile = reinterpret_cast<double*>(anb_smem + 2 * kAnbS * kTileBytes);  // [kAnbS][NB][448]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(
      anb_smem + 2 * kAnbS * kTileBytes + (size_t)kAnbS * NB * kAnbChunk * 8);

  const int wk = work[blockIdx.x];
  const int m = wk >> 16, rb = wk & 0xffff;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int b0 = blockIdx.y * NB;
  const int nbv = nb - b0 < NB ? nb - b0 : NB;
  const int L = T + 1;
  const int r0m = rowoff[m];
  const int rows = rowoff[m + 1] - r0m;
  const int le = n_even[m];
  const int rblock = r0m + rb * kTmaRows;
  const int rw = rb * kTmaRows + warp * kRowsPerWarp;
  const bool live = rw < rows;
  const bool ev0 = rw < le, ev1 = rw + 8 < le;
  const int nchunks = J / kTmaLat;
  const double* gsrc = reinterpret_cast<const double*>(gan) + ((size_t)b0 * L + m) * J * 28;
  const size_t bstride = (size_t)L * J * 28;  // doubles per state

  auto issue_tables = [&](int ch) {  // thread 0
    const int st = ch % kAnbS;
    mbar_expect_tx(&full[st], 2 * kTileBytes + nbv * kAnbChunk * 8);
    tma_load_2d(ptile + st * kTmaRows * kTmaLat, &pmap, ch * kTmaLat, rblock, &full[st]);
    tma_load_2d(htile + st * kTmaRows * kTmaLat, &hmap, ch * kTmaLat, rblock, &full[st]);
  };
  auto issue_data = [&](int ch) {  // thread 0, after the producer grid completed
    const int st = ch % kAnbS;
    for (int c = 0; c < nbv; ++c)
      bulk_g2s(btile + (st * NB + c) * kAnbChunk, gsrc + c * bstride + (size_t)ch * kAnbChunk,
               kAnbChunk * 8, &full[st]);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kAnbS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int ch = 0; ch < kAnbS && ch < nchunks; ++ch) issue_tables(ch);
  SDCSW_PDL_WAIT();
  if (threadIdx.x == 0)
    for (int ch = 0; ch < kAnbS && ch < nchunks; ++ch) issue_data(ch);

  // lane offsets in a k-step's 112-double record: [S: P 4x8 | H 4x6][A: same].
  // P: one 8-column tile per state.  H: the 6 H columns of all states packed
  // into NHT = ceil(6 NB / 8) tiles (global H column 8 h + g = state s, column
  // k; NB = 5: 9 instead of 10 DMMA pairs per k-step); H sums are kept apart
  // and added to the P sums in the epilogue.
  constexpr int NHT = (6 * NB + 7) / 8;
  const int po = t * 8 + g;
  int hoff[NHT];
#pragma unroll
  for (int h = 0; h < NHT; ++h) {
    const int col = 8 * h + g, hs_ = col / 6;
    hoff[h] = hs_ < NB ? hs_ * kAnbChunk + 32 + t * 6 + (col - 6 * hs_) : -1;
  }
  const bool any_ev = ev0 || ev1, any_od = !ev0 || !ev1;
  double acc[2][NB][2], acch[2][NHT][2];
#pragma unroll
  for (int a = 0; a < 2; ++a) {
#pragma unroll
    for (int c = 0; c < NB; ++c) acc[a][c][0] = acc[a][c][1] = 0.0;
#pragma unroll
    for (int h = 0; h < NHT; ++h) acch[a][h][0] = acch[a][h][1] = 0.0;
  }
  const int row0 = warp * kRowsPerWarp + g;

  for (int ch = 0; ch < nchunks; ++ch) {
    const int st = ch % kAnbS;
    mbar_wait(&full[st], (ch / kAnbS) & 1);
    if (live) {
      const double* pt = ptile + st * kTmaRows * kTmaLat;
      const double* ht = htile + st * kTmaRows * kTmaLat;
      const double* bt = btile + st * NB * kAnbChunk;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = 4 * q + t;
        const double aP0 = swz(pt, row0, k), aP1 = swz(pt, row0 + 8, k);
        const double aH0 = swz(ht, row0, k), aH1 = swz(ht, row0 + 8, k);
        double ps[NB], pa[NB], hs[NHT], ha[NHT];
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          const double* r = bt + c * kAnbChunk + q * 112;
          ps[c] = any_ev ? r[po] : 0.0;
          pa[c] = any_od ? r[56 + po] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < NHT; ++h) {
          const double* r = bt + q * 112 + (hoff[h] < 0 ? 0 : hoff[h]);
          hs[h] = any_od && hoff[h] >= 0 ? r[0] : 0.0;
          ha[h] = any_ev && hoff[h] >= 0 ? r[56] : 0.0;
        }
#pragma unroll
        for (int c = 0; c < NB; ++c) {
          dmma_t(acc[0][c], aP0, ev0 ? ps[c] : pa[c]);
          dmma_t(acc[1][c], aP1, ev1 ? ps[c] : pa[c]);
        }
#pragma unroll
        for (int h = 0; h < NHT; ++h) {
          dmma_t(acch[0][h], aH0, ev0 ? ha[h] : hs[h]);
          dmma_t(acch[1][h], aH1, ev1 ? ha[h] : hs[h]);
        }
      }
    }
    __syncthreads();  // every warp is done with stage st
    if (threadIdx.x == 0 && ch + kAnbS < nchunks) {
      issue_tables(ch + kAnbS);
      issue_data(ch + kAnbS);
    }
  }
  if (!live) return;
  double* o = ptile + warp * kRowsPerWarp * OS;  // P and H stages; all copies landed and were consumed
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int c = 0; c < NB; ++c) {
      o[(8 * a + g) * OS + 8 * c + 2 * t] = acc[a][c][0];
      o[(8 * a + g) * OS + 8 * c + 2 * t + 1] = acc[a][c][1];
    }
  __syncwarp();
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int h = 0; h < NHT; ++h) {  // columns (2t, 2t + 1) of H tile h: one state, one slot
      const int col = 8 * h + 2 * t, hs_ = col / 6;
      if (hs_ < NB) {
        double* d = o + (8 * a + g) * OS + 8 * hs_ + (col - 6 * hs_);
        d[0] += acch[a][h][0];
        d[1] += acch[a][h][1];
      }
    }
  __syncwarp();
  const int mo = moff[m];
  for (int it = lane; it < kRowsPerWarp * NB; it += 32) {
    const int rr = it % kRowsPerWarp, b = it / kRowsPerWarp;
    if (rw + rr >= rows || b0 + b >= nb) continue;
    const int n = row_n[r0m + rw + rr];
    if (n < 0) continue;
    const int idx = mo + n - m;
    const double* row = o + rr * OS;
    const double l = lam[idx];
    double2 phi = make_double2(row[8 * b + 0], row[8 * b + 1]);
    double2 zeta = make_double2(row[8 * b + 2], row[8 * b + 3]);
    double2 delta = make_double2(__fma_rn(l, row[8 * b + 6], row[8 * b + 4]),
                                 __fma_rn(l, row[8 * b + 7], row[8 * b + 5]));
    if (m == 0) phi.y = zeta.y = delta.y = 0.0;
    double2* dst = fe + (size_t)(b0 + b) * 3 * C;
    dst[idx] = phi;
    dst[C + idx] = zeta;
    dst[2 * C + idx] = delta;
  }
}

static_assert(kRowsPerWarp * (8 * 6 + 1) * 4 * 8 <= 2 * kAnbS * kTileBytes,
              "bulk analysis epilogue tiles fit in the table stage buffers");

cudaError_t configure_analysis_bulk() {
  cudaError_t e = cudaSuccess;
#define SDCSW_ANAB_CFG(NBV)                                                                   \
  if (e == cudaSuccess)                                                                       \
    e = cudaFuncSetAttribute(k_analysis_bulk<NBV>, cudaFuncAttributeMaxDynamicSharedMemorySize, \
                             (int)anab_smem<NBV>());
  SDCSW_ANAB_CFG(1) SDCSW_ANAB_CFG(2) SDCSW_ANAB_CFG(3) SDCSW_ANAB_CFG(4) SDCSW_ANAB_CFG(5)
  SDCSW_ANAB_CFG(6)
#undef SDCSW_ANAB_CFG
  return e;
}

static cudaError_t launch_analysis_bulk(const Plan& p, const Work& w, double2* fe, int nb,
                                        int NB, const int* work, int nwork, cudaStream_t s) {
  dim3 grid(nwork, (nb + NB - 1) / NB);
  const CUtensorMap& pm = *reinterpret_cast<const CUtensorMap*>(&p.tmap[0]);
  const CUtensorMap& hm = *reinterpret_cast<const CUtensorMap*>(&p.tmap[1]);
#define SDCSW_ANAB_LAUNCH(NBV)                                                                    \
  if (NB == NBV)                                                                                  \
    return launch_k(k_analysis_bulk<NBV>, grid, dim3(128), anab_smem<NBV>(), s, pm, hm, w.gan, nb, \
                    p.T, p.J, p.C, p.rowoff, p.n_even, p.row_n, p.moff, p.lam, work, fe);
  SDCSW_ANAB_LAUNCH(1) SDCSW_ANAB_LAUNCH(2) SDCSW_ANAB_LAUNCH(3) SDCSW_ANAB_LAUNCH(4)
  SDCSW_ANAB_LAUNCH(5) SDCSW_ANAB_LAUNCH(6)
#undef SDCSW_ANAB_LAUNCH
  return cudaErrorInvalidValue;
}


// ---------------------------------------------------------------------------
// H-free table-streaming analysis (legendre_ponly.cu): the five analysis data
// slots (A, B, C, D, E, folded and weighted by the ring kernel) of every state
// contracted with P only, for the degrees k = m..T+1 of the extended triangle:
//   ghat[b][(m, k)][slot] = sum_j P_k(mu_j) D_fold(k)[j, slot]
// (fold S for k - m even, A for odd).  Same TMA table stream and staged B
// operand as k_analysis_bulk, one table instead of two, and the 10 columns of
// each state packed into ceil(10 NB / 8) B tiles (NB = 5: 7 DMMA pairs per
// k-step instead of 9).  The i m factors and the H recurrence are applied by
// the assembly kernel (legendre_ponly.cu), which needs degrees k - 1 and k + 1.
// ---------------------------------------------------------------------------
constexpr int kAnpChunk = kTmaLat * kGanP;  // five-slot data doubles per state per stage
template <int NB>
constexpr size_t anap_smem() {
  return (size_t)kAnbS * (kTileBytes + NB * kAnpChunk * 8) + 8 * kAnbS;
}

template <int NB>
__global__ void __launch_bounds__(128, SDCSW_ANAB_MINB) k_analysis_bulk_ponly(
    const __grid_constant__ CUtensorMap pmap, const double* __restrict__ gan, int nb, int T, int J,
    const int* __restrict__ rowoff, const int* __restrict__ n_even, const int* __restrict__ row_n,
    const int* __restrict__ moffp, const int* __restrict__ work, double* __restrict__ ghat,
    int CP) {
  SDCSW_PDL_ENTRY();
  constexpr int NC = kGhat * NB;      // B columns: 10 per state
  constexpr int NT = (NC + 7) / 8;    // B tiles
  constexpr int OS = NC + 1;
  static_assert(kRowsPerWarp * OS * 4 * 8 <= kAnbS * (kTileBytes + NB * kAnpChunk * 8),
                "the epilogue tiles fit in the consumed stage buffers");
  extern __shared__ __align__(1024) unsigned char anp_smem[];
  double* ptile = reinterpret_cast<double*>(anp_smem);  // [kAnbS][64][16], swizzled
  double* btile = reinterpret_cast<double*>(anp_smem + kAnbS * kTileBytes);  // [kAnbS][NB][320]
  unsigned long long* full = reinterpret_cast<unsigned long long*>(
      anp_smem + kAnbS * kTileBytes + (size_t)kAnbS * NB * kAnpChunk * 8);

  const int wk = work[blockIdx.x];
  const int m = wk >> 16, rb = wk & 0xffff;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int g = lane >> 2, t = lane & 3;
  const int b0 = blockIdx.y * NB;
  const int nbv = nb - b0 < NB ? nb - b0 : NB;
  const int L = T + 1;
  const int r0m = rowoff[m];
  const int rows = rowoff[m + 1] - r0m;
  const int le = n_even[m];
  const int rblock = r0m + rb * kTmaRows;
  const int rw = rb * kTmaRows + warp * kRowsPerWarp;
  const bool live = rw < rows;
  const bool ev0 = rw < le, ev1 = rw + 8 < le;
  const int nchunks = J / kTmaLat;
  const double* gsrc = gan + ((size_t)b0 * L + m) * J * kGanP;
  const size_t bstride = (size_t)L * J * kGanP;  // doubles per state

  auto issue_tables = [&](int ch) {  // thread 0
    const int st = ch % kAnbS;
    mbar_expect_tx(&full[st], kTileBytes + nbv * kAnpChunk * 8);
    tma_load_2d(ptile + st * kTmaRows * kTmaLat, &pmap, ch * kTmaLat, rblock, &full[st]);
  };
  auto issue_data = [&](int ch) {  // thread 0, after the producer grid completed
    const int st = ch % kAnbS;
    for (int c = 0; c < nbv; ++c)
      bulk_g2s(btile + (st * NB + c) * kAnpChunk, gsrc + c * bstride + (size_t)ch * kAnpChunk,
               kAnpChunk * 8, &full[st]);
  };

  if (threadIdx.x == 0) {
    for (int s = 0; s < kAnbS; ++s) mbar_init(&full[s], 1);
    asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
  }
  __syncthreads();
  if (threadIdx.x == 0)
    for (int ch = 0; ch < kAnbS && ch < nchunks; ++ch) issue_tables(ch);
  SDCSW_PDL_WAIT();
  if (threadIdx.x == 0)
    for (int ch = 0; ch < kAnbS && ch < nchunks; ++ch) issue_data(ch);

  // B column 8 h + g of tile h = state s, double d of its 10 (5 slots x re, im);
  // per k-step (4 latitudes) a state's record is [fold][4 lat][10] = 80 doubles
  int boff[NT];
#pragma unroll
  for (int h = 0; h < NT; ++h) {
    const int col = 8 * h + g, s_ = col / kGhat;
    boff[h] = s_ < NB ? s_ * kAnpChunk + t * kGhat + (col - kGhat * s_) : -1;
  }
  const bool any_ev = ev0 || ev1, any_od = !ev0 || !ev1;
  double acc[2][NT][2];
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int h = 0; h < NT; ++h) acc[a][h][0] = acc[a][h][1] = 0.0;
  const int row0 = warp * kRowsPerWarp + g;

  for (int ch = 0; ch < nchunks; ++ch) {
    const int st = ch % kAnbS;
    mbar_wait(&full[st], (ch / kAnbS) & 1);
    if (live) {
      const double* pt = ptile + st * kTmaRows * kTmaLat;
      const double* bt = btile + st * NB * kAnpChunk;
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        const int k = 4 * q + t;
        const double aP0 = swz(pt, row0, k), aP1 = swz(pt, row0 + 8, k);
        double bs[NT], ba[NT];
#pragma unroll
        for (int h = 0; h < NT; ++h) {
          const double* r = bt + q * 80 + (boff[h] < 0 ? 0 : boff[h]);
          bs[h] = any_ev && boff[h] >= 0 ? r[0] : 0.0;
          ba[h] = any_od && boff[h] >= 0 ? r[40] : 0.0;
        }
#pragma unroll
        for (int h = 0; h < NT; ++h) {
          dmma_t(acc[0][h], aP0, ev0 ? bs[h] : ba[h]);
          dmma_t(acc[1][h], aP1, ev1 ? bs[h] : ba[h]);
        }
      }
    }
    __syncthreads();  // every warp is done with stage st
    if (threadIdx.x == 0 && ch + kAnbS < nchunks) {
      issue_tables(ch + kAnbS);
      issue_data(ch + kAnbS);
    }
  }
  if (!live) return;
  double* o = reinterpret_cast<double*>(anp_smem) + warp * kRowsPerWarp * OS;  // stages are consumed
#pragma unroll
  for (int a = 0; a < 2; ++a)
#pragma unroll
    for (int h = 0; h < NT; ++h) {
      const int col = 8 * h + 2 * t;
      if (col < NC) {
        o[(8 * a + g) * OS + col] = acc[a][h][0];
        o[(8 * a + g) * OS + col + 1] = acc[a][h][1];
      }
    }
  __syncwarp();
  const int mo = moffp[m];
  for (int it = lane; it < kRowsPerWarp * NB; it += 32) {
    const int rr = it % kRowsPerWarp, b = it / kRowsPerWarp;
    if (rw + rr >= rows || b0 + b >= nb) continue;
    const int k = row_n[r0m + rw + rr];
    if (k < 0) continue;
    const double* src = o + rr * OS + kGhat * b;
    double2* dst = reinterpret_cast<double2*>(ghat + ((size_t)(b0 + b) * CP + mo + k - m) * kGhat);
#pragma unroll
    for (int q = 0; q < kSlotsP; ++q) dst[q] = make_double2(src[2 * q], src[2 * q + 1]);
  }
}


cudaError_t configure_analysis_bulk_ponly() {
  cudaError_t e = cudaSuccess;
#define SDCSW_ANAP_CFG(NBV)                                                                   \
  if (e == cudaSuccess)                                                                       \
    e = cudaFuncSetAttribute(k_analysis_bulk_ponly<NBV>,                                      \
                             cudaFuncAttributeMaxDynamicSharedMemorySize, (int)anap_smem<NBV>());
  SDCSW_ANAP_CFG(1) SDCSW_ANAP_CFG(2) SDCSW_ANAP_CFG(3) SDCSW_ANAP_CFG(4) SDCSW_ANAP_CFG(5)
  SDCSW_ANAP_CFG(6)
#undef SDCSW_ANAP_CFG
  return e;
}

cudaError_t launch_analysis_bulk_ponly(const Plan& p, const Work& w, int nb, cudaStream_t s) {
  const int NB = nb <= 6 ? nb : 6;
  const bool own = p.own_idx != nullptr;  // split plan: own wavenumbers only
  const int* work = own ? p.own_workP : p.anal_workP;
  const int nwork = own ? p.n_own_workP : p.n_anal_workP;
  if (nwork < 1) return cudaSuccess;
  dim3 grid(nwork, (nb + NB - 1) / NB);
  const CUtensorMap& pm = *reinterpret_cast<const CUtensorMap*>(p.tmapP);
#define SDCSW_ANAP_LAUNCH(NBV)                                                                   \
  if (NB == NBV)                                                                                 \
    return launch_k(k_analysis_bulk_ponly<NBV>, grid, dim3(128), anap_smem<NBV>(), s, pm,         \
                    reinterpret_cast<const double*>(w.gan), nb, p.T, p.J, p.rowoffP, p.n_evenP,  \
                    p.rowP_n, p.moffP, work, w.ghat, p.CP);
  SDCSW_ANAP_LAUNCH(1) SDCSW_ANAP_LAUNCH(2) SDCSW_ANAP_LAUNCH(3) SDCSW_ANAP_LAUNCH(4)
  SDCSW_ANAP_LAUNCH(5) SDCSW_ANAP_LAUNCH(6)
#undef SDCSW_ANAP_LAUNCH
  return cudaErrorInvalidValue;
}

// TMA map over the H-free table [rowsP][J] (same box and swizzle as the P/H maps)
cudaError_t make_table_map_ponly(Plan& p) {
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  cudaError_t e = cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q);
  if (e != cudaSuccess || !fn || q != cudaDriverEntryPointSuccess) return cudaErrorNotSupported;
  auto encode = reinterpret_cast<PFN_cuTensorMapEncodeTiled>(fn);
  const cuuint64_t dims[2] = {(cuuint64_t)p.J, (cuuint64_t)p.rowsP + 16};
  const cuuint64_t strides[1] = {(cuuint64_t)p.J * sizeof(double)};
  const cuuint32_t box[2] = {kTmaLat, kTmaRows};
  const cuuint32_t elem[2] = {1, 1};
  CUresult r = encode(reinterpret_cast<CUtensorMap*>(p.tmapP), CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2,
                      p.ptabP, dims, strides, box, elem, CU_TENSOR_MAP_INTERLEAVE_NONE,
                      CU_TENSOR_MAP_SWIZZLE_128B, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
                      CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS ? cudaSuccess : cudaErrorNotSupported;
}

}  // namespace sdcsw
