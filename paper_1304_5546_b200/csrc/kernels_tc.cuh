// fp32 stage kernels on the 5th-generation tensor cores (tcgen05.mma kind::tf32, TMEM).
// Included by kernels.cuh when DG_MMA == 3 (fp32).  DESIGN.md §6 "tcgen05 path".
//
// A CTA (4 warps, 128 threads) owns a GROUP of TG = 4 consecutive 32-element tiles: the MMA's
// M = 128 rows are the group's elements, thread t <-> element t <-> TMEM lane t (warp w reads and
// writes lanes 32w..32w+31).  Per group and stage (eq. 9 with readings A1/A2, 1/2 eq. 5 flux, A12):
//
//   volume (H2):  the CUDA cores write the A operands into TMEM (tcgen05.st), one row per element:
//                 Ez and W1 = rx Hy - ry Hx, W2 = sx Hy - sy Hx (K = nodes), each split into tf32
//                 hi + lo; one thread issues
//                   [u | v] (N = 2 Np)  = Ez [Dr^T | Ds^T]          (D columns C_U .. C_V + Np)
//                   w       (N = Np)    = W1 Dr^T + W2 Ds^T          (D columns C_W ..)
//                 as 3xTF32 products (lo*hi + hi*lo + hi*hi), B operands (the operators, hi and lo)
//                 in shared memory.
//   flux (H3-H4): per face point of its element each thread forms the Fsc-scaled flux (fHx, fHy,
//                 fEz) and maps the H part through the inverse chain rule,
//                   [gx, gy] = G^-1 [fHx, fHy],  G = [[-ry, -sy], [rx, sx]],  G^-1 = J [[sx, sy], [-rx, -ry]],
//                 so that the LIFT can accumulate into the SAME accumulators as the volume term:
//   lift (H5):    u += gx LIFT^T,  v += gy LIFT^T,  w += fEz LIFT^T   (K = 3 Nfp face points),
//                 and then  rhsHx = -(ry u + sy v) = -Dy Ez + LIFT fHx,  rhsHy = rx u + sx v,
//                 rhsEz = w   (G (u + LIFT g) = G u + LIFT f: the chain rule is linear, G per element).
//   update (H6):  tcgen05.ld of u, v, w -> 1/mu, 1/eps -> LSERK4 (res, q_out) with coalesced stores.
// Fields, geometry and the LSERK4 residual keep the tile-blocked layout of kernel_api.h with the
// identity column swizzle (every smem access is one element per lane: conflict free).
#pragma once

namespace tc {

// DG_TCP: the neighbour codes of group it+1 are loaded into registers while group it computes, so
// the traces' loads at the top of a group do not first wait for their codes
#ifndef DG_TCP
#define DG_TCP 1
#endif
// DG_TCR: the L2 prefetch of a group (one ahead) also covers its LSERK4 residual (measured 6% slower: off)
#ifndef DG_TCR
#define DG_TCR 0
#endif
// DG_TCE: the LSERK4 residual of the whole group loaded at its top (see the group loop)
#ifndef DG_TCE
#define DG_TCE 0
#endif
constexpr bool TCE = DG_TCE;
constexpr int TG = 4;                    // tiles per group
constexpr int MG = TG * TL;              // MMA M = 128 elements
// DG_TH threads per element (1 or 2): thread (element e, half h) owns columns 8k + CW h .. + CW - 1 of
// every 8-column chunk of the A operands, the face points and the output nodes (CW = 8 / DG_TH)
#ifndef DG_TH
#define DG_TH 2
#endif
constexpr int NH = DG_TH;
static_assert(NH == 1 || NH == 2, "DG_TH");
constexpr int CW = 8 / NH;
constexpr int NTH = MG * NH;             // threads per CTA
constexpr int NPN = 8 * ((NP + 7) / 8);  // accumulator columns per field (MMA N, granularity 8)
constexpr int NPK = NPN;                 // volume K padding (k-steps of 8 tf32)
constexpr int NFK = 8 * ((NF + 7) / 8);  // LIFT K padding
constexpr int KSV = NPK / 8, KSL = NFK / 8;
constexpr int AK = NPK > NFK ? NPK : NFK;  // columns per A sub-block
// TMEM columns: accumulators u | v | w, then six A sub-blocks (hi/lo of three operands)
constexpr int C_U = 0, C_V = NPN, C_W = 2 * NPN;
constexpr int C_A = ((3 * NPN + 15) / 16) * 16;
constexpr int TM_NEED = C_A + 6 * AK;
static_assert(TM_NEED <= 512, "TMEM budget");
constexpr int TM_COLS = TM_NEED <= 32 ? 32 : TM_NEED <= 64 ? 64 : TM_NEED <= 128 ? 128 : TM_NEED <= 256 ? 256 : 512;
constexpr int TM_CTAS = 512 / TM_COLS;   // resident CTAs per SM the TMEM allows
// B operands in shared memory: K-major, no swizzle, 8-row x 16-byte core matrices
//   offset(n, k) = (k/8) KSTEP + ((k%8)/4) LBO + (n/8) 128 + (n%8) 16 + (k%4) 4
// BV: [Dr^T rows 0..NPN) | Ds^T rows NPN..2NPN)] x K = NPK;  BL: LIFT^T NPN rows x K = NFK
constexpr uint32_t LBO_V = (2 * NPN / 8) * 128, KST_V = 2 * LBO_V, SZ_BV = KSV * KST_V;
constexpr uint32_t LBO_L = (NPN / 8) * 128, KST_L = 2 * LBO_L, SZ_BL = KSL * KST_L;
constexpr size_t OPS = 2 * (size_t)SZ_BV + 2 * (size_t)SZ_BL;  // BV hi, BV lo, BL hi, BL lo
constexpr size_t QF = (size_t)TG * NP * TL * 4;                 // one field of a group
__host__ __device__ constexpr size_t GB_(bool mat) { return (size_t)TG * (mat ? dg::NGEO_MAT : dg::NGEO_CONST) * TL * 4; }
constexpr size_t BARS = 64;
// two {q, geo} buffers (group t+1 streams in while t computes) when they fit in 227 KB, else one
__host__ __device__ constexpr size_t buf_bytes(bool mat) { return 3 * QF + GB_(mat); }
__host__ __device__ constexpr int nbuf(bool mat) { return BARS + OPS + 2 * buf_bytes(mat) <= 227 * 1024 ? 2 : 1; }
__host__ __device__ constexpr size_t smem_bytes(bool mat) { return BARS + OPS + nbuf(mat) * buf_bytes(mat); }
// residual kept in registers between the LIFT issue and the epilogue when small enough
constexpr bool RES_REGS = 3 * 8 * ((NP + 7) / 8) / NH <= 84;
// register cap: two 4-warp CTAs per SM need <= 232 registers per thread (the occupancy
// calculator rejects 248 x 256 threads); one CTA per SM (512 TMEM columns) may use 255
#ifndef DG_TC_MAXREG
#define DG_TC_MAXREG (NH == 2 ? 128 : 232)
#endif
constexpr int TC_MAXREG = TM_CTAS >= 2 ? DG_TC_MAXREG : (NH == 2 ? 255 : 255);

__host__ __device__ constexpr uint32_t idesc(int n) {  // kind::tf32, fp32 D, K-major A and B, M = 128
  return (1u << 4) | (2u << 7) | (2u << 10) | ((uint32_t)(n >> 3) << 17) | ((uint32_t)(MG >> 4) << 24);
}
__device__ __forceinline__ uint64_t sdesc(uint32_t saddr, uint32_t lbo) {  // SWIZZLE_NONE, SBO = 128 B
  return (uint64_t)((saddr >> 4) & 0x3FFF) | ((uint64_t)((lbo >> 4) & 0x3FFF) << 16) |
         ((uint64_t)(128 >> 4) << 32) | ((uint64_t)1 << 46);
}
__device__ __forceinline__ void mma(uint32_t d, uint32_t a, uint64_t b, uint32_t id, uint32_t acc) {
  asm volatile(
      "{\n.reg .pred p;\nsetp.ne.b32 p, %4, 0;\n"
      "tcgen05.mma.cta_group::1.kind::tf32 [%0], [%1], %2, %3, p;\n}\n" ::"r"(d),
      "r"(a), "l"(b), "r"(id), "r"(acc)
      : "memory");
}
__device__ __forceinline__ void commit(uint64_t* bar) {
  asm volatile("tcgen05.commit.cta_group::1.mbarrier::arrive::one.shared::cluster.b64 [%0];\n" ::"r"(smem_u32(bar))
               : "memory");
}
__device__ __forceinline__ void st8(uint32_t taddr, const uint32_t (&v)[8]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x8.b32 [%0], {%1,%2,%3,%4,%5,%6,%7,%8};\n" ::"r"(taddr), "r"(v[0]),
               "r"(v[1]), "r"(v[2]), "r"(v[3]), "r"(v[4]), "r"(v[5]), "r"(v[6]), "r"(v[7])
               : "memory");
}
__device__ __forceinline__ void ld8(uint32_t taddr, float (&v)[8]) {
  uint32_t r[8];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x8.b32 {%0,%1,%2,%3,%4,%5,%6,%7}, [%8];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3]), "=r"(r[4]), "=r"(r[5]), "=r"(r[6]), "=r"(r[7])
               : "r"(taddr)
               : "memory");
#pragma unroll
  for (int j = 0; j < 8; ++j) v[j] = __uint_as_float(r[j]);
}
__device__ __forceinline__ void fence_before() { asm volatile("tcgen05.fence::before_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void fence_after() { asm volatile("tcgen05.fence::after_thread_sync;\n" ::: "memory"); }
__device__ __forceinline__ void wait_st() { asm volatile("tcgen05.wait::st.sync.aligned;\n" ::: "memory"); }
__device__ __forceinline__ void wait_ld() { asm volatile("tcgen05.wait::ld.sync.aligned;\n" ::: "memory"); }

__device__ __forceinline__ void st4(uint32_t taddr, const uint32_t (&v)[4]) {
  asm volatile("tcgen05.st.sync.aligned.32x32b.x4.b32 [%0], {%1,%2,%3,%4};\n" ::"r"(taddr), "r"(v[0]), "r"(v[1]),
               "r"(v[2]), "r"(v[3])
               : "memory");
}
__device__ __forceinline__ void ld4(uint32_t taddr, float (&v)[4]) {
  uint32_t r[4];
  asm volatile("tcgen05.ld.sync.aligned.32x32b.x4.b32 {%0,%1,%2,%3}, [%4];\n"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(taddr)
               : "memory");
#pragma unroll
  for (int j = 0; j < 4; ++j) v[j] = __uint_as_float(r[j]);
}
// this thread's CW columns of TMEM (32x32b: its lane) <-> registers
__device__ __forceinline__ void st_cols(uint32_t taddr, const uint32_t (&v)[8]) { st8(taddr, v); }
__device__ __forceinline__ void st_cols(uint32_t taddr, const uint32_t (&v)[4]) { st4(taddr, v); }
__device__ __forceinline__ void ld_cols(uint32_t taddr, float (&v)[8]) { ld8(taddr, v); }
__device__ __forceinline__ void ld_cols(uint32_t taddr, float (&v)[4]) { ld4(taddr, v); }
// x = hi + lo (split_tf32 of kernels.cuh): CW values -> the hi and lo A sub-blocks
__device__ __forceinline__ void st_split(uint32_t thi, uint32_t tlo, const float (&x)[CW]) {
  uint32_t hi[CW], lo[CW];
#pragma unroll
  for (int j = 0; j < CW; ++j) split_tf32(x[j], hi[j], lo[j]);
  st_cols(thi, hi);
  st_cols(tlo, lo);
}

// The MMA chains of one group (issued by one thread).  Passes per k-step: (A lo, B hi),
// (A hi, B lo), (A hi, B hi) -- the 3xTF32 product; the first MMA into an accumulator overwrites.
__device__ __forceinline__ void issue_volume(uint32_t tm, uint32_t ops) {
  constexpr uint32_t IDV = idesc(2 * NPN), IDN = idesc(NPN);
  const uint32_t bv[2] = {ops, ops + SZ_BV};  // hi, lo
#pragma unroll
  for (int ks = 0; ks < KSV; ++ks)
#pragma unroll
    for (int pass = 0; pass < 3; ++pass) {
      const int ah = pass == 0 ? 1 : 0;  // A sub-block offset: 0 hi, 1 lo
      const uint32_t b = bv[pass == 1 ? 1 : 0] + ks * KST_V;
      const uint32_t first = (ks == 0 && pass == 0) ? 0u : 1u;
      mma(tm + C_U, tm + C_A + (0 + ah) * AK + 8 * ks, sdesc(b, LBO_V), IDV, first);
      mma(tm + C_W, tm + C_A + (2 + ah) * AK + 8 * ks, sdesc(b, LBO_V), IDN, first);
      mma(tm + C_W, tm + C_A + (4 + ah) * AK + 8 * ks, sdesc(b + (NPN / 8) * 128, LBO_V), IDN, 1u);
    }
}
__device__ __forceinline__ void issue_lift(uint32_t tm, uint32_t ops, bool accumulate) {
  constexpr uint32_t IDN = idesc(NPN);
  const uint32_t bl[2] = {ops + 2 * SZ_BV, ops + 2 * SZ_BV + SZ_BL};
#pragma unroll
  for (int ks = 0; ks < KSL; ++ks)
#pragma unroll
    for (int pass = 0; pass < 3; ++pass) {
      const int ah = pass == 0 ? 1 : 0;
      const uint64_t b = sdesc(bl[pass == 1 ? 1 : 0] + ks * KST_L, LBO_L);
      const uint32_t acc = (accumulate || ks > 0 || pass > 0) ? 1u : 0u;
      mma(tm + C_U, tm + C_A + (0 + ah) * AK + 8 * ks, b, IDN, acc);
      mma(tm + C_V, tm + C_A + (2 + ah) * AK + 8 * ks, b, IDN, acc);
      mma(tm + C_W, tm + C_A + (4 + ah) * AK + 8 * ks, b, IDN, acc);
    }
}

template <int MODE, bool MAT>
__global__ void __maxnreg__(TC_MAXREG) stage_kernel_tc(const dg::StageArgs p) {
  using MT = ModeTraits<MODE>;
  constexpr int NG = MAT ? dg::NGEO_MAT : dg::NGEO_CONST;
  constexpr size_t GB = GB_(MAT);
  constexpr size_t BUF = 3 * QF + GB;  // one {q, geo} buffer
  constexpr int NB = nbuf(MAT);
  constexpr int FS = TG * NP * TL;     // field stride of a group in shared memory (elements)
  constexpr int KC = KSL * CW;         // face points per thread
  extern __shared__ __align__(128) unsigned char smem_raw[];
  uint64_t* bar_tma = reinterpret_cast<uint64_t*>(smem_raw);  // [2]: one per {q, geo} buffer
  uint64_t* bar_mma = bar_tma + 2;
  uint32_t* tm_slot = reinterpret_cast<uint32_t*>(smem_raw + 32);
  unsigned char* sops = smem_raw + BARS;
  auto sq_of = [&](int it) { return reinterpret_cast<float*>(sops + OPS + (it % NB) * BUF); };
  auto sg_of = [&](int it) { return reinterpret_cast<float*>(sops + OPS + (it % NB) * BUF + 3 * QF); };
  const float* __restrict__ q = static_cast<const float*>(p.q_in);
  const float* __restrict__ geo = static_cast<const float*>(p.geo);
  // thread -> (element e of the group = TMEM lane, column half h); tile-in-group ti = warp % 4
  const int tid = threadIdx.x, e = tid % MG, h = tid / MG, ti = e >> 5, lane = tid & 31;
  const int first = blockIdx.x, stride = gridDim.x;
  const int n_it = first < p.ntiles ? (p.ntiles - first + stride - 1) / stride : 0;
  if (n_it == 0) return;
  const bool read_res = MT::rk && p.a != 0.0;
  auto group_of = [&](int it) {
    const int sidx = first + it * stride;
    const int j = p.reverse ? p.ntiles - 1 - sidx : sidx;
    return p.tiles ? p.tiles[j] : j;
  };
  auto point = [&](int kk) { return 8 * (kk / CW) + CW * h + kk % CW; };  // face point of slot kk
  auto issue_tma = [&](int it) {
    if (tid == 0) {
      const int64_t g = group_of(it);
      uint64_t* bar = bar_tma + (it % NB);
      mbar_expect_tx(bar, (unsigned)BUF);
      float* sq = sq_of(it);
#pragma unroll
      for (int c = 0; c < 3; ++c) tma_load_1d(sq + c * FS, q + c * p.fstride + g * FS, (unsigned)QF, bar);
      tma_load_1d(sg_of(it), geo + g * TG * NG * TL, (unsigned)GB, bar);
    }
  };
  auto prefetch_l2 = [&](int it) {  // fields, geometry and neighbour codes of group `it`
    if (tid == 0) {
      const int64_t g = group_of(it);
#pragma unroll
      for (int c = 0; c < 3; ++c) bulk_prefetch_l2(q + c * p.fstride + g * FS, (unsigned)QF);
      bulk_prefetch_l2(geo + g * TG * NG * TL, (unsigned)GB);
      if (MT::surf) bulk_prefetch_l2(p.vmapP + g * TG * NF * TL, (unsigned)(TG * NF * TL * 4));
      if (DG_TCR && MT::rk && p.a != 0.0) {  // the LSERK4 residual the epilogue reads (DG_TCR)
        const float* res = static_cast<const float*>(p.res);
#pragma unroll
        for (int c = 0; c < 3; ++c) bulk_prefetch_l2(res + c * p.vstride + g * FS, (unsigned)QF);
      }
    }
  };

  // prologue: barriers, operators (B hi/lo blocks, once per persistent CTA), TMEM
  if (tid == 0) {
    mbar_init(bar_tma, 1);
    mbar_init(bar_tma + 1, 1);
    mbar_init(bar_mma, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  {
    const int4* src = reinterpret_cast<const int4*>(p.ops);
    int4* dst = reinterpret_cast<int4*>(sops);
    for (int i = tid; i < (int)(OPS / 16); i += NTH) dst[i] = __ldg(src + i);
  }
  asm volatile("fence.proxy.async.shared::cta;\n" ::: "memory");  // generic writes -> MMA operand reads
  if (tid < 32) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;\n" ::"r"(smem_u32(tm_slot)),
                 "r"(TM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;\n");
  }
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tm = *tm_slot;
  const uint32_t tml = tm + ((uint32_t)(32 * ti) << 16) + CW * h;  // lane quarter, column half
  const uint32_t ops_s = smem_u32(sops);

  issue_tma(0);
  if (n_it > 1) prefetch_l2(1);
  uint32_t mma_par = 0;
  const float alpha = static_cast<float>(p.alpha);
#ifdef DG_TC_PROF
  long long ph[12] = {}, tp = clock64();
  auto mark = [&](int k) { if (tid == 0 || tid == 32) { const long long t = clock64(); ph[k] += t - tp; tp = t; } };
#else
  auto mark = [](int) {};
#endif

  int32_t vcn[KC];
  auto load_codes = [&](int it2, int32_t (&v)[KC]) {
    const int32_t* src = p.vmapP + (group_of(it2) * TG + ti) * NF * TL + lane;
#pragma unroll
    for (int kk = 0; kk < KC; ++kk) v[kk] = point(kk) < NF ? __ldg(src + point(kk) * TL) : -1;
  };
  if (DG_TCP && MT::surf) load_codes(0, vcn);
  for (int it = 0; it < n_it; ++it) {
    const int64_t grp = group_of(it);
    // neighbour codes of this thread's face points (L2: prefetched one group ahead), then the
    // cross-group neighbour traces straight into registers -- in flight during the volume phase
    int32_t vc[KC];
    float nb[3][KC];
    if constexpr (MT::surf) {
      if constexpr (DG_TCP) {
#pragma unroll
        for (int kk = 0; kk < KC; ++kk) vc[kk] = vcn[kk];
      } else {
        load_codes(it, vc);
      }
#pragma unroll
      for (int kk = 0; kk < KC; ++kk)
#pragma unroll
        for (int c = 0; c < 3; ++c) nb[c][kk] = vc[kk] >= 0 ? __ldg(q + vc[kk] + c * p.fstride) : 0.f;
      if (DG_TCP && it + 1 < n_it) load_codes(it + 1, vcn);
    }
    mbar_wait(bar_tma + (it % NB), (unsigned)((it / NB) & 1));
    mark(0);
    __syncthreads();  // also: every thread is done with buffer (it + 1) & 1 (group it - 1)
    mark(1);
    if (NB == 2 && it + 1 < n_it) issue_tma(it + 1);
    if (NB == 1 && it + 1 < n_it) prefetch_l2(it + 1);  // its TMA is issued after this group
    if (NB == 2 && it + 2 < n_it) prefetch_l2(it + 2);
    // DG_TCE: the whole LSERK4 residual of this thread's nodes is loaded here, in flight during the
    // volume and flux phases, instead of one 8-node chunk ahead inside the epilogue
    float rall[TCE ? KSV : 1][3][CW];
    if constexpr (TCE && MT::rk) {
      if (read_res) {
        const int64_t tb0 = ((grp * TG + ti) * NP) * TL + lane;
        const float* __restrict__ res0 = static_cast<const float*>(p.res);
#pragma unroll
        for (int ks = 0; ks < KSV; ++ks)
#pragma unroll
          for (int j = 0; j < CW; ++j) {
            const int n = 8 * ks + CW * h + j;
            const int64_t o = tb0 + (n < NP ? n : NP - 1) * TL;
#pragma unroll
            for (int c = 0; c < 3; ++c) rall[ks][c][j] = __ldcs(res0 + c * p.vstride + o);
          }
      }
    }
    const float* sq = sq_of(it);
    const float* gg = sg_of(it) + ti * NG * TL + lane;  // this element's geometry column
    const float rx = gg[0 * TL], sx = gg[1 * TL], ry = gg[2 * TL], sy = gg[3 * TL];
    float imu = 1.f, ieps = 1.f;
    if constexpr (MAT) {
      if (MODE != dg::MODE_VOLUME || p.scale_volume) {
        imu = gg[16 * TL];
        ieps = gg[17 * TL];
      }
    }
    const float* sqe = sq + ti * NP * TL + lane;  // node n of field c: sqe[c * FS + n * TL]

    // ---- volume operands (this thread's CW columns of every 8-column chunk) -> TMEM, volume MMAs
    if constexpr (MT::vol) {
#pragma unroll
      for (int ks = 0; ks < KSV; ++ks) {
        float ez[CW], w1[CW], w2[CW];
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          const int n = 8 * ks + CW * h + j;
          if (n < NP) {
            const float hx = sqe[n * TL], hy = sqe[FS + n * TL];
            ez[j] = sqe[2 * FS + n * TL];
            w1[j] = rx * hy - ry * hx;
            w2[j] = sx * hy - sy * hx;
          } else {
            ez[j] = w1[j] = w2[j] = 0.f;
          }
        }
        st_split(tml + C_A + 0 * AK + 8 * ks, tml + C_A + 1 * AK + 8 * ks, ez);
        st_split(tml + C_A + 2 * AK + 8 * ks, tml + C_A + 3 * AK + 8 * ks, w1);
        st_split(tml + C_A + 4 * AK + 8 * ks, tml + C_A + 5 * AK + 8 * ks, w2);
      }
      wait_st();
      fence_before();
      mark(2);
      __syncthreads();
      mark(3);
      if (tid == 0) {
        fence_after();
        issue_volume(tm, ops_s);
        commit(bar_mma);
      }
      mark(4);
    }

    // ---- flux of this thread's face points (registers), then LIFT operands -> TMEM
    if constexpr (MT::surf) {
      float fx[KC], fy[KC], fz[KC];
      const float J = 1.f / (rx * sy - ry * sx);  // det G = rx sy - ry sx = 1/J (affine element)
#pragma unroll
      for (int kk = 0; kk < KC; ++kk) {
        const int m = point(kk);
        fx[kk] = fy[kk] = fz[kk] = 0.f;
        if (m < NF) {
          const int f = m / NFP, i = m - f * NFP;
          const int fm = fmask(f, i);
          const float nx = gg[(4 + 3 * f) * TL], ny = gg[(5 + 3 * f) * TL], hF = gg[(6 + 3 * f) * TL];
          const float bsc = gg[(13 + f) * TL];
          const int code = vc[kk];
          float pHx = nb[0][kk], pHy = nb[1][kk], pEz = nb[2][kk];
          if (code < 0) {  // neighbour in this group: shared memory
            const float* pp = sq + (-1 - code);
            pHx = pp[0];
            pHy = pp[FS];
            pEz = pp[2 * FS];
          }
          const float dHx = sqe[fm * TL] - pHx;
          const float dHy = sqe[FS + fm * TL] - pHy;
          const float dEz = sqe[2 * FS + fm * TL] - bsc * pEz;
          float fHx, fHy, fEz;
          if constexpr (!MAT) {
            const float ndotdH = nx * dHx + ny * dHy;
            fHx = hF * (ny * dEz + alpha * (nx * ndotdH - dHx));
            fHy = hF * (-nx * dEz + alpha * (ny * ndotdH - dHy));
            fEz = hF * (ny * dHx - nx * dHy - alpha * dEz);
          } else {
            const float wEH = gg[(18 + 4 * f) * TL], wHH = gg[(19 + 4 * f) * TL];
            const float wHE = gg[(20 + 4 * f) * TL], wEE = gg[(21 + 4 * f) * TL];
            const float dHt = nx * dHy - ny * dHx;
            const float gH = wEH * dEz + wHH * dHt;
            fHx = hF * (ny * gH);
            fHy = -hF * (nx * gH);
            fEz = -hF * (wHE * dHt + wEE * dEz);
          }
          fx[kk] = J * (sx * fHx + sy * fHy);   // G^-1 [fHx, fHy]
          fy[kk] = -J * (rx * fHx + ry * fHy);
          fz[kk] = fEz;
        }
      }
      mark(5);
      if constexpr (MT::vol) {  // the volume MMAs must be done reading the A region
        mbar_wait(bar_mma, mma_par);
        mma_par ^= 1u;
        fence_after();
      }
      mark(6);
#pragma unroll
      for (int ks = 0; ks < KSL; ++ks) {
        float a[CW], b[CW], c[CW];
#pragma unroll
        for (int j = 0; j < CW; ++j) {
          a[j] = fx[ks * CW + j];
          b[j] = fy[ks * CW + j];
          c[j] = fz[ks * CW + j];
        }
        st_split(tml + C_A + 0 * AK + 8 * ks, tml + C_A + 1 * AK + 8 * ks, a);
        st_split(tml + C_A + 2 * AK + 8 * ks, tml + C_A + 3 * AK + 8 * ks, b);
        st_split(tml + C_A + 4 * AK + 8 * ks, tml + C_A + 5 * AK + 8 * ks, c);
      }
      wait_st();
      fence_before();
      mark(7);
      __syncthreads();
      if (tid == 0) {
        fence_after();
        issue_lift(tm, ops_s, MT::vol);
        commit(bar_mma);
      }
      mark(8);
    }

    // ---- epilogue: the residual of this thread's nodes into registers (one chunk ahead) while the
    // MMAs finish; u, v, w out of TMEM; LSERK4 update with q_in from shared memory
    const int64_t tb = ((grp * TG + ti) * NP) * TL + lane;  // element's node-0 offset in a field
    const float* __restrict__ resin = static_cast<const float*>(p.res);
    auto load_res = [&](int ks, float (&rv)[3][CW]) {
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int n = 8 * ks + CW * h + j;
        const int64_t o = tb + (n < NP ? n : NP - 1) * TL;
#pragma unroll
        for (int c = 0; c < 3; ++c) rv[c][j] = (MT::rk && read_res) ? __ldcs(resin + c * p.vstride + o) : 0.f;
      }
    };
    float ra[3][CW], rb[3][CW];
    if constexpr (!TCE) load_res(0, ra);
    mark(9);
    mbar_wait(bar_mma, mma_par);
    mma_par ^= 1u;
    fence_after();
    mark(10);
    const float a = static_cast<float>(p.a), b = static_cast<float>(p.b), dt = static_cast<float>(p.dt);
#pragma unroll
    for (int ks = 0; ks < KSV; ++ks) {
      float (&rv)[3][CW] = TCE ? rall[TCE ? ks : 0] : ((ks & 1) ? rb : ra);
      if (!TCE && ks + 1 < KSV) {
        if (ks & 1) load_res(ks + 1, ra);
        else load_res(ks + 1, rb);
      }
      float u[CW], v[CW], z[CW];
      ld_cols(tml + C_U + 8 * ks, u);
      ld_cols(tml + C_V + 8 * ks, v);
      ld_cols(tml + C_W + 8 * ks, z);
      wait_ld();
#pragma unroll
      for (int j = 0; j < CW; ++j) {
        const int n = 8 * ks + CW * h + j;
        if (n >= NP) break;
        float rhs[3] = {-(ry * u[j] + sy * v[j]), rx * u[j] + sx * v[j], z[j]};
        const int64_t o = tb + n * TL;
        if constexpr (MODE == dg::MODE_SURFACE_RK) {
          const float* __restrict__ rvs = static_cast<const float*>(p.rhsv);
#pragma unroll
          for (int c = 0; c < 3; ++c) rhs[c] += rvs[c * p.vstride + o];
        }
        if constexpr (MAT) {
          rhs[0] *= imu;
          rhs[1] *= imu;
          rhs[2] *= ieps;
        }
        if constexpr (MT::rk) {
          float* __restrict__ res = static_cast<float*>(p.res);
          float* __restrict__ qo = static_cast<float*>(p.q_out);
#pragma unroll
          for (int c = 0; c < 3; ++c) {
            float rs = dt * rhs[c];
            if (read_res) rs = fmaf(a, rv[c][j], rs);
            if (p.write_res) st_out(res + c * p.vstride + o, rs);
            st_out(qo + c * p.fstride + o, fmaf(b, rs, sqe[c * FS + n * TL]));
          }
        } else {
          float* __restrict__ out = static_cast<float*>(p.out);
#pragma unroll
          for (int c = 0; c < 3; ++c) out[c * p.vstride + o] = rhs[c];
        }
      }
    }
    fence_before();  // D is rewritten by the next group's first MMA after the next barrier
    mark(11);
    if (NB == 1 && it + 1 < n_it) {  // one buffer: the next group's loads after every thread is done
      __syncthreads();
      issue_tma(it + 1);
    }
  }
#ifdef DG_TC_PROF
  if ((tid == 0 || tid == 32) && blockIdx.x == 0 && p.a != 0.0)
    printf("tc prof tid %d (%d groups): tma %lld | bar %lld | volop %lld | bar %lld | mmaissue %lld | flux %lld | "
           "volwait %lld | fluxop %lld | bar+issue %lld | resld %lld | liftwait %lld | epi %lld\n",
           tid, n_it, ph[0], ph[1], ph[2], ph[3], ph[4], ph[5], ph[6], ph[7], ph[8], ph[9], ph[10], ph[11]);
#endif
  __syncthreads();
  if (tid < 32) asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;\n" ::"r"(tm), "r"(TM_COLS));
}

template <int MODE, bool MAT>
cudaError_t launch_one(const dg::StageArgs& a, cudaStream_t s) {
  constexpr size_t smem = smem_bytes(MAT);
  static int grid_cap[64] = {0};
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  if (e != cudaSuccess) return e;
  if (dev >= 64) return cudaErrorInvalidDevice;
  if (grid_cap[dev] == 0) {
    e = cudaFuncSetAttribute(stage_kernel_tc<MODE, MAT>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
    if (e != cudaSuccess) return cudaGetLastError(), e;
    // all of the unified L1/shared array as shared memory: two 82 KB CTAs per SM (the default
    // carve-out preference leaves the occupancy calculator at one)
    e = cudaFuncSetAttribute(stage_kernel_tc<MODE, MAT>, cudaFuncAttributePreferredSharedMemoryCarveout,
                             (int)cudaSharedmemCarveoutMaxShared);
    if (e != cudaSuccess) return e;
    // resident CTAs per SM from the kernel's own limits: TMEM columns, shared memory (+1 KB
    // reserved per CTA), registers.  (cudaOccupancyMaxActiveBlocksPerMultiprocessor answers 1 for
    // this kernel whatever its registers and shared memory -- measured: 0.243 ms per C4 stage at two
    // CTAs per SM against 0.354 ms at the calculator's one.)
    cudaFuncAttributes fa{};
    e = cudaFuncGetAttributes(&fa, stage_kernel_tc<MODE, MAT>);
    if (e != cudaSuccess) return e;
    int sms = 0, smem_sm = 0, regs_sm = 0;
    if ((e = cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev)) != cudaSuccess) return e;
    if ((e = cudaDeviceGetAttribute(&smem_sm, cudaDevAttrMaxSharedMemoryPerMultiprocessor, dev)) != cudaSuccess)
      return e;
    if ((e = cudaDeviceGetAttribute(&regs_sm, cudaDevAttrMaxRegistersPerMultiprocessor, dev)) != cudaSuccess)
      return e;
    const int by_smem = smem_sm / (int)(smem + fa.sharedSizeBytes + 1024);
    const int regs_warp = ((fa.numRegs * 32 + 255) / 256) * 256;
    const int by_regs = regs_sm / (regs_warp * (NTH / 32));
    int per_sm = TM_CTAS < by_smem ? TM_CTAS : by_smem;
    if (by_regs < per_sm) per_sm = by_regs;
    grid_cap[dev] = (per_sm > 0 ? per_sm : 1) * sms;
  }
  int grid = a.ntiles < grid_cap[dev] ? a.ntiles : grid_cap[dev];
  if (a.max_ctas > 0 && grid > a.max_ctas) grid = a.max_ctas;
  if (grid <= 0) return cudaSuccess;
  stage_kernel_tc<MODE, MAT><<<grid, NTH, smem, s>>>(a);
  return cudaGetLastError();
}

// Host: operators into the B blocks (hi = tf32(x), lo = tf32(x - hi); padded rows/columns zero)
inline void pack(const double* Dr, const double* Ds, const double* LIFT, unsigned char* o) {
  auto hi_of = [](double x) {
    const float f = static_cast<float>(x);
    uint32_t u;
    std::memcpy(&u, &f, 4);
    u = (u + 0x1000u) & 0xFFFFE000u;
    float h;
    std::memcpy(&h, &u, 4);
    return h;
  };
  auto put = [&](size_t base, uint32_t lbo, int n, int k, double x) {
    const size_t off = (size_t)(k / 8) * (2 * lbo) + ((k % 8) / 4) * lbo + (n / 8) * 128 + (n % 8) * 16 + (k % 4) * 4;
    const float h = hi_of(x), l = hi_of(x - (double)h);
    std::memcpy(o + base + off, &h, 4);
    std::memcpy(o + base + off + (base < 2 * SZ_BV ? SZ_BV : SZ_BL), &l, 4);
  };
  std::memset(o, 0, OPS);
  for (int n = 0; n < NP; ++n)
    for (int k = 0; k < NP; ++k) {
      put(0, LBO_V, n, k, Dr[n * NP + k]);        // B[n][k] = Dr[n][k]: D[e][n] = sum_k A[e][k] Dr[n][k]
      put(0, LBO_V, NPN + n, k, Ds[n * NP + k]);
    }
  for (int n = 0; n < NP; ++n)
    for (int m = 0; m < NF; ++m) put(2 * SZ_BV, LBO_L, n, m, LIFT[n * NF + m]);
}

}  // namespace tc
