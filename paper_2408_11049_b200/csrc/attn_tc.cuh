// attn_tc.cuh — the tcgen05 (5th-generation tensor core) verify kernel, included by attn.cu
// after the stream-K machinery (AttnParams, Plan, SegWalker, finish_unit) it reuses.
//
// md_verify_attn_full for R = g*(gamma+1) in (8, 128] query rows per KV head at head_dim 128
// (GQA verify: Llama-3.1 R = 20, Qwen2.5 R = 35; up to gamma = 15 with g = 8, or Qwen2.5 (g = 7)
// to gamma = 15 = 112 rows; SURVEY §8(a) row a3, §8(b) g*T <= 128).  Swapped operands so
// the tensor-core work is 2 * 128 * NP FLOP per key (NP = R rounded up to 16), not 128 rows:
//   S^T[128 keys][NP]  = K[128 keys][d] . Q^T            (A = K tile, K-major SW128 from TMA;
//                                                          B = Q rows, K-major SW128 from TMA)
//   O^T[d][NP]        += V^T . P^T                       (A = V tile read MN-major, SW128;
//                                                          B = P^T, MN-major 8x8 core matrices)
// Both accumulators live in TMEM (S^T double-buffered by tile, O^T by segment: 4 NP <= 512
// columns).  Warp roles (1 CTA / SM, 3 x 64 KB K/V stages of 128 keys; 2 stages above NP = 48):
//   warp 4NG    TMA producer: the segment's Q rows (one 3-D box per 64-column slab) and K/V tiles;
//   warp 4NG+1  MMA issuer (one thread) + TMEM allocator: S^T(i) is issued before PV(i-1);
//   warps 0..4NG-1 softmax + epilogue in NG row groups of 4 warps (NG = 1 up to NP = 48, else
//           NP / 32 groups of 32 rows), thread x of a group <-> TMEM lane x (key x of the tile
//           for S^T, head dim x for O^T): each thread owns one key's scores for the group's rows, so the online softmax needs
//           no cross-thread work per tile except a CTA vote: the running row maxima m are only
//           raised when a score exceeds m + 8 (log2 units; P stays <= 2^8, exact in the
//           fp32 sums and a bf16 operand like any other), which rescales the thread-local row
//           sums and O^T in TMEM (tcgen05.ld/st); row sums are reduced across the 128 threads
//           once per segment.  Keys past the tile's valid range get P = 0 and their V rows
//           are zeroed in shared memory (fetched cache rows past kv_len may hold NaN bits).
// Stream-K decomposition, split partials and the fused last-arriver merge are those of the
// mma.sync kernels (64-key plan tiles; a 128-key stage covers two of them).

#include <type_traits>

namespace tc {  // helpers: tcgen05.cuh (included by attn.cu)

constexpr int KT = 128;                      // keys per stage (MMA M)
constexpr int SLAB = KT * 128;               // one 64-column slab of a 128-key tile
constexpr int STAGE = 4 * SLAB;              // K (2 slabs) + V (2 slabs) = 64 KB
constexpr float THR = 8.f;                   // lazy max-raise threshold (log2 units)
constexpr int SMEM_MAX = 232448;             // 227 KB per CTA

// NP = R rounded up to 16 query-row columns (<= 128: S^T x2 + O^T x2 = 4 NP <= 512 TMEM columns).
// Up to 48 columns one group of 128 softmax threads holds every row's state in registers; above
// that the rows are cut into NG = 2 groups of CW = NP / 2 columns, each group a further 4 warps
// over the same 128 TMEM lanes (warp w reads lane quadrant w % 4), which walk their columns in
// chunks of CH = 32 (or 16) in two passes per stage (max test, then exponentials), so a thread
// keeps only its CW row sums and one chunk of scores.
#ifndef MD_TC_CH16
#define MD_TC_CH16 0  // A/B: 16-column TMEM chunks for every row-group width
#endif
template <int NP>
struct Cfg {
  static constexpr int NG = NP <= 48 ? 1 : 2;        // row groups
  static constexpr int CW = NP / NG;                 // query-row columns per group
  static constexpr int CH = (CW == 32 && !MD_TC_CH16) ? 32 : 16;  // columns per TMEM load chunk (NG > 1)
  static constexpr int SM_THREADS = 128 * NG;        // softmax / epilogue threads
  static constexpr int THREADS = SM_THREADS + 64;    // + producer warp + MMA warp
  static constexpr int NQ = NP <= 32 ? 2 : 1;        // Q buffers (by segment parity)
  static constexpr int QBUF = 2 * NP * 128;          // Q rows, two 64-column SW128 slabs
  static constexpr int PBUF = NP * KT * 2;           // P^T, 8x8 core matrices
  static constexpr int HDR = 384;                    // barriers, tmem slot, flags, plan
  static constexpr int AUX = HDR + 6 * NP * 4;       // + red[4NG][CW], mrow[NP], crow[NP]
  // the dynamic shared memory starts 1 KB aligned (no static __shared__; checked at entry)
  static constexpr int FIXED = NQ * QBUF + PBUF + AUX + TABLE_BYTES;
  static constexpr int NSTAGE = (3 * STAGE + FIXED <= SMEM_MAX) ? 3 : 2;
  static constexpr int SMEM = NSTAGE * STAGE + FIXED;
  static constexpr int TMEM_COLS = 4 * NP <= 128 ? 128 : (4 * NP <= 256 ? 256 : 512);
  static_assert(NP % 16 == 0 && NP >= 16 && NP <= 128, "16 <= NP <= 128, a multiple of 16");
  static_assert(NG == 1 || CW % 16 == 0, "group columns in whole 16-column loads");
  static_assert(SMEM <= SMEM_MAX, "shared memory budget");
};

// OR-vote over the 128 softmax threads of a row group (named barrier `id`)
__device__ __forceinline__ bool vote_any128(bool v, int id = 2) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred q, p;\n\tsetp.ne.u32 q, %1, 0;\n\tbarrier.cta.red.or.pred p, %2, 128, q;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)v), "r"(id)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ void bar128(int id = 2) { named_bar_sync(id, 128); }

// diagnostics (md_debug_trace): cycles spent in a wait, accumulated by one thread
__device__ __forceinline__ void twait(uint64_t* bar, uint32_t parity, long long* acc) {
  if (acc == nullptr) {
    mbar_wait(bar, parity);
    return;
  }
  const long long t0 = clock64();
  mbar_wait(bar, parity);
  *acc += clock64() - t0;
}

// stages of a segment: [lo*64, min(keys, hi*64)) in 128-key steps
__device__ __forceinline__ int seg_stages(const Ranges& rg) { return (rg.e0 - rg.s0 + KT - 1) / KT; }

// TMA producer (one thread): Q rows of the segment, then its K/V stages.  K and V halves of a
// stage have their own full / empty barriers: the K half is free once the tile's S^T MMAs
// complete, the V half only after its PV, so the next K loads go out a whole softmax earlier.
// The V half of tile i is issued after the K half of tile i + 1 (V is consumed one softmax
// later than K), so a K load never waits behind the longer V release.
#ifndef MD_TC_PF
#define MD_TC_PF 0  // measured: 2 or 4 stages of L2 prefetch slow Llama verify 1.26 -> 1.41 ms
#endif
constexpr int PF = MD_TC_PF;  // stages prefetched into L2 ahead of the ring
struct PendV {                // a V half not yet issued
  int it, pos, nvalid, b, kvh;
};
__device__ __forceinline__ int half_bytes(int nvalid) {  // bytes of one K (or V) half
  int bytes = 0;
  for (int h = 0; h < 2; ++h) {
    const int hv = nvalid - h * TK;
    if (hv >= TK) bytes += 2 * TK * 128;
    else if (hv > 0) bytes += 2 * ((hv + BOX_ROWS - 1) / BOX_ROWS) * BOX_ROWS * 128;
  }
  return bytes;
}
template <int NSTAGE>
__device__ __forceinline__ void load_half(const CUtensorMap* full_map, const CUtensorMap* part_map, uint8_t* dst,
                                          uint64_t* bar, int pos, int nvalid, int kvh, int b, uint64_t pol) {
  for (int h = 0; h < 2; ++h) {
    const int hv = nvalid - h * TK, r0 = pos + h * TK;
    for (int sub = 0; sub < 2; ++sub) {
      const int off = sub * SLAB + h * TK * 128;
      if (hv >= TK) {
        tma_load_4d(dst + off, full_map, bar, sub * 64, r0, kvh, b, pol);
      } else if (hv > 0) {
        for (int bx = 0; bx * BOX_ROWS < hv; ++bx)
          tma_load_4d(dst + off + bx * BOX_ROWS * 128, part_map, bar, sub * 64, r0 + bx * BOX_ROWS, kvh, b, pol);
      }
    }
  }
}
template <int NSTAGE>
__device__ __forceinline__ void issue_v(const TmapSet& tm, uint8_t* ring, uint64_t* vfull, uint64_t* vempty,
                                        const PendV& pv, uint64_t pol) {
  const int stage = pv.it % NSTAGE;
  mbar_wait(&vempty[stage], ((pv.it / NSTAGE) & 1) ^ 1);
  mbar_arrive_expect_tx(&vfull[stage], half_bytes(pv.nvalid));
  load_half<NSTAGE>(&tm.v_full, &tm.v_part, ring + stage * STAGE + 2 * SLAB, &vfull[stage], pv.pos, pv.nvalid, pv.kvh,
                    pv.b, pol);
}
template <int NP>
__device__ void produce(const AttnParams& p, const TmapSet& tm, const CUtensorMap* qmap, const Seg& sg,
                        const Ranges& rg, uint8_t* ring, uint8_t* qbuf, uint64_t* full, uint64_t* empty,
                        uint64_t* vfull, uint64_t* vempty, uint64_t* qfull, uint64_t* qempty, int& it, int& qi,
                        PendV& pend, uint64_t pol, long long* tw, uint64_t* apb) {
  using C = Cfg<NP>;
  const int qs = qi % C::NQ;
  mbar_wait(&qempty[qs], ((qi / C::NQ) & 1) ^ 1);
  mbar_arrive_expect_tx(&qfull[qs], 2 * p.R * 128);
  for (int sub = 0; sub < 2; ++sub)
    tma_load_4d(qbuf + qs * C::QBUF + sub * NP * 128, qmap, &qfull[qs], sub * 64, sg.kvh * p.g, 0, sg.b, pol);
  ++qi;
  for (int pos = rg.s0; pos < rg.e0; pos += KT, ++it) {
    const int stage = it % C::NSTAGE;
    const int nvalid = min(KT, rg.e0 - pos);
    if (tile_has_new(p, sg.n, pos, nvalid)) mbar_wait(apb, 0);  // fused append done
    twait(&empty[stage], ((it / C::NSTAGE) & 1) ^ 1, tw);
    mbar_arrive_expect_tx(&full[stage], half_bytes(nvalid));
    // L2 prefetch PF stages ahead (full 64-row boxes only)
    if (PF > 0) {
      const int pp = pos + PF * KT;
      for (int h = 0; h < 2; ++h) {
        const int r0 = pp + h * TK;
        if (r0 + TK <= rg.e0)
          for (int sub = 0; sub < 2; ++sub) {
            tma_prefetch_4d(&tm.k_full, sub * 64, r0, sg.kvh, sg.b);
            tma_prefetch_4d(&tm.v_full, sub * 64, r0, sg.kvh, sg.b);
          }
      }
    }
    load_half<C::NSTAGE>(&tm.k_full, &tm.k_part, ring + stage * STAGE, &full[stage], pos, nvalid, sg.kvh, sg.b, pol);
    if (pend.it >= 0) issue_v<C::NSTAGE>(tm, ring, vfull, vempty, pend, pol);
    pend = PendV{it, pos, nvalid, sg.b, sg.kvh};
  }
}

// Zero key x's V row of a stage (cache rows past the valid keys may hold NaN bits).  The 16-byte
// chunks are visited in a lane-rotated order, so the 8 lanes of a quarter-warp store to 8
// different bank groups (the rows are 128 bytes apart: the same chunk order would be 8-way).
__device__ __forceinline__ void zero_vrow(uint8_t* vrow, int x) {
#pragma unroll
  for (int c = 0; c < 8; ++c) {
    const int cc = (c + x) & 7;
    *reinterpret_cast<uint4*>(vrow + cc * 16) = make_uint4(0, 0, 0, 0);
    *reinterpret_cast<uint4*>(vrow + SLAB + cc * 16) = make_uint4(0, 0, 0, 0);
  }
}

// RR > 0: the row count R is a compile-time constant (the hot configurations), else p.R
template <int NP, int RR>
__global__ void __launch_bounds__(Cfg<NP>::THREADS, 1)
    attn_tc_kernel(const __grid_constant__ TmapSet tm, const __grid_constant__ CUtensorMap qmap, const AttnParams p) {
  using C = Cfg<NP>;
  constexpr int NG = C::NG, CW = C::CW, SM_THREADS = C::SM_THREADS;
  const int R = RR > 0 ? RR : p.R;
  constexpr int NSTAGE = C::NSTAGE, NQ = C::NQ;
  constexpr int D = 128;
  extern __shared__ __align__(1024) uint8_t smem_raw[];
  // SWIZZLE_128B tiles need 1 KB alignment: the dynamic window follows the 1 KB reserved block
  // (no static shared memory), so it is aligned; the budget keeps no slack for realignment
  if (smem_u32(smem_raw) & 1023u) __trap();
  uint8_t* smem = smem_raw;
  uint8_t* ring = smem;
  uint8_t* qbuf = ring + NSTAGE * STAGE;
  uint8_t* pbuf = qbuf + NQ * C::QBUF;
  uint64_t* full = reinterpret_cast<uint64_t*>(pbuf + C::PBUF);
  uint64_t* empty = full + NSTAGE;
  uint64_t* qfull = empty + NSTAGE;  // [2]
  uint64_t* qempty = qfull + 2;      // [2]
  uint64_t* sfull = qempty + 2;      // [2]
  uint64_t* sempty = sfull + 2;      // [2]
  uint64_t* pfull = sempty + 2;      // [1]
  uint64_t* pempty = pfull + 1;      // [1]
  uint64_t* ofull = pempty + 1;      // [2]
  uint64_t* oempty = ofull + 2;      // [2]
  uint64_t* vfull = oempty + 2;      // [NSTAGE] V halves of the ring stages (full / empty: K halves)
  uint64_t* vempty = vfull + NSTAGE; // [NSTAGE]
  uint64_t* apb = vempty + NSTAGE;   // [1] fused append: the group-0 softmax warps' new-row stores are done
  uint32_t* tslot = reinterpret_cast<uint32_t*>(apb + 1);
  int* flag = reinterpret_cast<int*>(tslot + 4);                 // [16] finish_unit
  Plan* plan_smem = reinterpret_cast<Plan*>(flag + 16);          // 40 bytes (reserved 64)
  static_assert((4 * NSTAGE + 15) * 8 + 16 + 64 + 64 <= C::HDR, "barrier / flag header");
  float* red = reinterpret_cast<float*>(smem + NSTAGE * STAGE + NQ * C::QBUF + C::PBUF + C::HDR);  // [4NG][CW]
  float* mrow = red + 4 * NP;                                    // [NP] running row maxima (log2 units)
  float* crow = mrow + NP;                                       // [NP] rescale factors / row sums
  int* pre = reinterpret_cast<int*>(crow + NP);                  // [TABLE_B + 1]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  constexpr int PRODUCER = 4 * NG, ISSUER = 4 * NG + 1;  // warp roles after the softmax warps
  if (threadIdx.x == 0) {
    for (int s = 0; s < NSTAGE; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], 1);
      mbar_init(&vfull[s], 1);
      mbar_init(&vempty[s], 1);
    }
    for (int s = 0; s < 2; ++s) {
      mbar_init(&qfull[s], 1);
      mbar_init(&qempty[s], 1);
      mbar_init(&sfull[s], 1);
      mbar_init(&sempty[s], 4 * NG);
      mbar_init(&ofull[s], 1);
      mbar_init(&oempty[s], 4 * NG);
    }
    mbar_init(pfull, 4 * NG);
    mbar_init(pempty, 1);
    mbar_init(apb, 4);
    fence_mbar_init();
  }
  // Q rows >= R stay zero for the whole kernel (the TMA boxes write rows < R only)
  for (int i = threadIdx.x; i < NQ * C::QBUF / 16; i += C::THREADS) {
    const int slab_row = (i * 16 / 128) % NP;
    if (slab_row >= p.R) reinterpret_cast<uint4*>(qbuf)[i] = make_uint4(0, 0, 0, 0);
  }
  fence_proxy_async();
  if (warp == ISSUER) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == PRODUCER && lane == 0) {  // descriptor fetches overlap the grid-dependency wait
    prefetch_tmap(&tm.k_full);
    prefetch_tmap(&tm.v_full);
    prefetch_tmap(&tm.k_part);
    prefetch_tmap(&tm.v_part);
    prefetch_tmap(&qmap);
  }
  if (p.pdl_early) pdl_trigger();
  pdl_wait();  // kv_len, the cache and q may come from the previous kernel
  fence_before();
  __syncthreads();
  fence_after();
  const uint32_t tbase = *tslot;
  build_prefix(p, pre);
  if (threadIdx.x == 0) *plan_smem = make_plan(p, total_tiles(p, pre), gridDim.x);
  __syncthreads();
  const Plan& pl = *plan_smem;  // static stream-K plan (the host sets dyn_k = 0 for this kernel)
  const int chunk = blockIdx.x;
  const bool active = (int)blockIdx.x < pl.G;
  SegWalker walk;
  Seg sg;
  if (active) {
    int64_t S0, E0;
    cta_range(p, pre, pl, chunk, S0, E0);
    walk.init(p, pre, S0, E0);
  }
  if (p.kn != nullptr && warp < 4 && active) {  // fused append: the new rows of this CTA's tiles
    int64_t S0, E0;
    cta_range(p, pre, pl, chunk, S0, E0);
    SegWalker aw;
    aw.init(p, pre, S0, E0);
    append_own_rows<128>(p, pre, aw, threadIdx.x, 128);
    __syncwarp();
    if (lane == 0) mbar_arrive(apb);
  }

  if (warp == PRODUCER) {
    // ============================== TMA producer ==============================
    if (active && lane == 0) {
      const uint64_t pol = policy_evict_first();
      int it = 0, qi = 0;
      PendV pend{-1, 0, 0, 0, 0};
      long long tw = 0;
      long long* twp = p.trace ? &tw : nullptr;
      while (walk.next(p, pre, sg))
        produce<NP>(p, tm, &qmap, sg, seg_ranges(p, sg), ring, qbuf, full, empty, vfull, vempty, qfull, qempty, it, qi,
                    pend, pol, twp, apb);
      if (pend.it >= 0) issue_v<NSTAGE>(tm, ring, vfull, vempty, pend, pol);
      if (p.trace) trace_put(p, 15, tw);
    }
  } else if (warp == ISSUER) {
    // ============================== MMA issuer ==============================
    if (active && lane == 0) {
      constexpr uint32_t ID_S = idesc(128, NP, 0, 0), ID_O = idesc(128, NP, 1, 1);
      const uint32_t ring_a = smem_u32(ring), q_a = smem_u32(qbuf), p_a = smem_u32(pbuf);
      int it = 0, tt = 0, qi = 0, si = 0;
      long long w_full = 0, w_se = 0, w_pf = 0;
      long long* wf = p.trace ? &w_full : nullptr;
      long long* ws_ = p.trace ? &w_se : nullptr;
      long long* wp = p.trace ? &w_pf : nullptr;
      // the PV of the previous tile is issued after this tile's S^T (S^T double-buffered)
      int pv_stage = -1, pv_ob = 0, pv_first = 0, pv_last = 0, pv_tt = 0, pv_it = 0;
      auto issue_pv = [&]() {
        mbar_wait(&vfull[pv_stage], (pv_it / NSTAGE) & 1);
        twait(pfull, pv_tt & 1, wp);
        fence_after();
        const uint32_t vt = ring_a + pv_stage * STAGE + 2 * SLAB;
        const uint32_t od = tbase + 2 * NP + pv_ob * NP;
#pragma unroll
        for (int kk = 0; kk < KT / 16; ++kk)
          mma_f16(od, sdesc(vt + kk * 2048, SLAB, 1024, 2), sdesc(p_a + kk * 256, 128, 2048, 0), ID_O,
                  (pv_first && kk == 0) ? 0u : 1u);
        commit(&vempty[pv_stage]);
        commit(pempty);
        if (pv_last) commit(&ofull[pv_ob]);
        pv_stage = -1;
      };
      while (walk.next(p, pre, sg)) {
        const Ranges rg = seg_ranges(p, sg);
        const int ns = seg_stages(rg);
        const int qs = qi % NQ, ob = si & 1;
        mbar_wait(&qfull[qs], (qi / NQ) & 1);
        mbar_wait(&oempty[ob], ((si >> 1) & 1) ^ 1);
        for (int j = 0; j < ns; ++j, ++it, ++tt) {
          const int stage = it % NSTAGE, sb = tt & 1;
          twait(&full[stage], (it / NSTAGE) & 1, wf);
          twait(&sempty[sb], ((tt >> 1) & 1) ^ 1, ws_);
          fence_after();
          const uint32_t kt = ring_a + stage * STAGE;
#pragma unroll
          for (int kk = 0; kk < D / 16; ++kk) {
            const uint32_t off = (kk >> 2) * SLAB + (kk & 3) * 32;
            const uint32_t qoff = (kk >> 2) * (NP * 128) + (kk & 3) * 32;
            mma_f16(tbase + sb * NP, sdesc(kt + off, 16, 1024, 2), sdesc(q_a + qs * C::QBUF + qoff, 16, 1024, 2), ID_S,
                    kk > 0 ? 1u : 0u);
          }
          commit(&sfull[sb]);
          commit(&empty[stage]);  // the K half is free once S^T is complete
          if (j == ns - 1) commit(&qempty[qs]);
          if (pv_stage >= 0) issue_pv();
          pv_stage = stage;
          pv_ob = ob;
          pv_first = (j == 0);
          pv_last = (j == ns - 1);
          pv_tt = tt;
          pv_it = it;
        }
        ++qi;
        ++si;
      }
      if (pv_stage >= 0) issue_pv();
      if (p.trace) {
        trace_put(p, 8, w_full);
        trace_put(p, 9, w_se);
        trace_put(p, 10, w_pf);
        trace_put(p, 11, tt);
      }
    }
  } else if (active && NG == 1) {
    // ====================== softmax + epilogue, all rows in one group (NP <= 48) ======================
    const int x = threadIdx.x;                      // TMEM lane: key of the tile / head-dim row of O^T
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    int it = 0, tt = 0, si = 0;
    long long w_sf = 0, w_pe = 0, w_epi = 0, t_start = clock64();
    long long* wsf = (p.trace && x == 0) ? &w_sf : nullptr;
    long long* wpe = (p.trace && x == 0) ? &w_pe : nullptr;
    float mr[NP], lacc[NP];
    while (walk.next(p, pre, sg)) {
      const int b = sg.b, kvh = sg.kvh, n = sg.n;
      const Ranges rg = seg_ranges(p, sg);
      const int ns = seg_stages(rg);
      const int ob = si & 1;
      const int vbase = n - p.T;
#pragma unroll
      for (int r = 0; r < NP; ++r) {
        mr[r] = -INFINITY;
        lacc[r] = 0.f;
      }
      if (x < NP) mrow[x] = -INFINITY;
      bar128();
      for (int j = 0; j < ns; ++j, ++it, ++tt) {
        const int stage = it % NSTAGE, sb = tt & 1;
        const int pos = rg.s0 + j * KT;
        const int nvalid = min(KT, rg.e0 - pos);
        const int key = pos + x;                    // cache position (verify)
        const bool valid = x < nvalid;
        twait(&sfull[sb], (tt >> 1) & 1, wsf);
        fence_after();
        float v[NP];
#pragma unroll
        for (int c = 0; c < NP; c += 16) tld16(tbase + sb * NP + c + lane_off, v + c);
        wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[sb]);
        // x_r = s_r * scale * log2(e) - m_r: one FMA per row, reused for the raise test and
        // the exponent.  Masking (keys past the valid range; the causal chain / tree mask among
        // the T new keys) only exists in a unit's last stage: a tile-uniform branch.
        const float sl2 = p.scale_log2;
        const bool edge = (nvalid < KT) || (pos + KT > vbase);
        const int rel = key - vbase;
        float xs[NP];
        float xmax = -INFINITY;
#pragma unroll
        for (int r = 0; r < NP; ++r) {
          xs[r] = (r < R) ? fmaf(v[r], sl2, -mr[r]) : -INFINITY;
          xmax = fmaxf(xmax, xs[r]);
        }
        if (edge) {
          // masked keys get x = -inf (also their scaled scores v = -inf for a max raise)
          uint32_t msk = p.tree_mask ? __ldg(p.tree_mask + (size_t)b * p.T) : 1u;
          int t = 0, hh = 0;
          xmax = -INFINITY;
#pragma unroll
          for (int r = 0; r < NP; ++r) {
            const bool hide = !valid || (rel >= 0 && !((msk >> (rel & 31)) & 1u));
            if (r < R && hide) xs[r] = -INFINITY;
            if (r < R && hide) v[r] = -INFINITY;
            xmax = fmaxf(xmax, xs[r]);
            if (++hh == p.g) {  // next query token t (row r = t * g + hh)
              hh = 0;
              ++t;
              if (t < p.T) msk = p.tree_mask ? __ldg(p.tree_mask + (size_t)b * p.T + t) : ((2u << t) - 1u);
            }
          }
        }
        const bool need = xmax > THR;  // some score exceeds its row maximum by > 2^8 (or m = -inf)
        // the previous tile's PV must be complete before P is rewritten or O^T rescaled
        if (tt > 0) twait(pempty, (tt - 1) & 1, wpe);
        if (vote_any128(need)) {
          // raise every row's maximum to this tile's (or keep it): per-row max over the tile
#pragma unroll
          for (int r = 0; r < NP; ++r) {
            if (r < R) {
              float m = (v[r] == -INFINITY) ? -INFINITY : v[r] * sl2;
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
              if (lane == 0) red[warp * NP + r] = m;
            }
          }
          bar128();
          if (x < R) {
            const float m = fmaxf(fmaxf(red[x], red[NP + x]), fmaxf(red[2 * NP + x], red[3 * NP + x]));
            const float mo = mrow[x];
            const float mn = fmaxf(mo, m);
            crow[x] = (mo == -INFINITY) ? 0.f : ex2(mo - mn);
            mrow[x] = mn;
          }
          bar128();
#pragma unroll
          for (int r = 0; r < NP; ++r) {
            if (r < R) {
              mr[r] = mrow[r];
              lacc[r] *= crow[r];
              const float base = (mr[r] == -INFINITY) ? 0.f : mr[r];
              xs[r] = (v[r] == -INFINITY) ? -INFINITY : fmaf(v[r], sl2, -base);
            }
          }
          if (j > 0) {  // O^T already holds PV of earlier tiles of this segment: rescale it
            const uint32_t oa = tbase + 2 * NP + ob * NP + lane_off;
#pragma unroll
            for (int c = 0; c < NP; c += 16) {
              float o[16];
              tld16(oa + c, o);
              wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] *= (c + i < R) ? crow[c + i] : 0.f;
              tst16(oa + c, o);
            }
            wait_st();
          }
        }
        // P = 2^x; row sums accumulate in fp32, the MMA operand is bf16
        uint32_t pk[NP / 2];
#pragma unroll
        for (int r = 0; r < NP; r += 2) {
          const float p0 = (r < R) ? ex2(xs[r]) : 0.f, p1 = (r + 1 < R) ? ex2(xs[r + 1]) : 0.f;
          lacc[r] += p0;
          lacc[r + 1] += p1;
          pk[r / 2] = pack_bf16(p0, p1);
        }
        // P^T core layout: key x -> core column x / 8, row (x % 8) * 16 B; rows r -> core r / 8
        uint8_t* pd = pbuf + (x >> 3) * 128 + (x & 7) * 16;
#pragma unroll
        for (int c = 0; c < NP / 8; ++c)
          *reinterpret_cast<uint4*>(pd + c * 2048) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        if (!valid) {  // zero this key's V row (after the V half's TMA writes land)
          mbar_wait(&vfull[stage], (it / NSTAGE) & 1);
          zero_vrow(ring + stage * STAGE + 2 * SLAB + x * 128, x);
        }
        fence_proxy_async();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(pfull);
      }
      // ---------------- segment epilogue: row sums over the 128 key lanes, O^T / l
      const long long t_epi = p.trace ? clock64() : 0;
#pragma unroll
      for (int r = 0; r < NP; ++r) {
        float l = lacc[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        if (lane == 0) red[warp * NP + r] = l;
      }
      bar128();
      if (x < NP) crow[x] = red[x] + red[NP + x] + red[2 * NP + x] + red[3 * NP + x];  // L_r
      mbar_wait(&ofull[ob], (si >> 1) & 1);
      fence_after();
      float o[NP];
#pragma unroll
      for (int c = 0; c < NP; c += 16) tld16(tbase + 2 * NP + ob * NP + c + lane_off, o + c);
      wait_ld();
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&oempty[ob]);
      bar128();
      const bool complete = sg.complete();
      const int slot_base = seg_slot(p, pl, sg, chunk);
#pragma unroll
      for (int r = 0; r < NP; ++r) {
        if (r < R) {
          const float L = crow[r];
          const float val = (L > 0.f) ? o[r] / L : 0.f;
          if (complete) store_out(p, o_row(p, b, kvh, r) * D + x, val);
          else __stcg(p.ws_o + ((int64_t)slot_base * p.R + r) * D + x, val);
        }
      }
      if (x < R) {
        const float L = crow[x], m = mrow[x];
        const float lse2 = (L > 0.f) ? m + __log2f(L) : -INFINITY;
        if (complete) {
          if (p.lse != nullptr) p.lse[out_row(p, b, kvh, x)] = lse2 * LN2;
        } else {
          __stcg(p.ws_lse + (int64_t)slot_base * p.R + x, lse2);
        }
      }
      if (!complete) finish_unit<D>(p, sg, pl, SM_THREADS, flag);
      bar128();  // red / mrow / crow reused by the next segment
      if (p.trace) w_epi += clock64() - t_epi;
      ++si;
    }
    if (p.trace && x == 0) {
      trace_put(p, 12, w_sf);
      trace_put(p, 13, w_pe);
      trace_put(p, 14, clock64() - t_start);
      trace_put(p, 7, w_epi);  // segment epilogues (row sums, O^T read, stores, split merge)
      trace_put(p, 6, globaltimer());  // softmax end (ns): the CTA's finish time
    }
  } else if (active) {
    // ===== softmax + epilogue, row group grp of NG = 2 (CW columns [cb, cb + CW), chunks of CH) =====
    constexpr int CH = C::CH, NCH = CW / CH;
    const int x = threadIdx.x & 127;                // TMEM lane: key of the tile / head-dim row of O^T
    const int grp = threadIdx.x >> 7, wq = warp & 3, cb = grp * CW;
    const int bar_id = 2 + grp;                     // the group's named barrier
    const uint32_t lane_off = (uint32_t)(wq * 32) << 16;
    float* gred = red + grp * 4 * CW;               // [4][CW] per-warp row partials of this group
    int it = 0, tt = 0, si = 0;
    float lacc[CW];
    auto tload = [&](uint32_t addr, float* v) {     // CH consecutive TMEM columns
#pragma unroll
      for (int c = 0; c < CH; c += 16) tld16(addr + c, v + c);
      wait_ld();
    };
    while (walk.next(p, pre, sg)) {
      const int b = sg.b, kvh = sg.kvh, n = sg.n;
      const Ranges rg = seg_ranges(p, sg);
      const int ns = seg_stages(rg);
      const int ob = si & 1;
      const int vbase = n - p.T;
#pragma unroll
      for (int r = 0; r < CW; ++r) lacc[r] = 0.f;
      if (x < CW) mrow[cb + x] = -INFINITY;
      bar128(bar_id);
      for (int j = 0; j < ns; ++j, ++it, ++tt) {
        const int stage = it % NSTAGE, sb = tt & 1;
        const int pos = rg.s0 + j * KT;
        const int nvalid = min(KT, rg.e0 - pos);
        const bool valid = x < nvalid;
        const bool edge = (nvalid < KT) || (pos + KT > vbase);
        const int rel = pos + x - vbase;
        const float sl2 = p.scale_log2;
        const uint32_t s_col = tbase + sb * NP + cb + lane_off;
        // dead(r): key x is invisible to query row cb + r (a padded row, a key past the valid
        // range, or a new key outside the row's causal chain / tree mask)
        uint64_t dead = 0;
        if (edge) {
#pragma unroll 1
          for (int r = 0; r < CW; ++r)
            if (cb + r >= R) dead |= 1ull << r;
          int t = cb / p.g, hh = cb - t * p.g;
          uint32_t msk = t < p.T ? (p.tree_mask ? __ldg(p.tree_mask + (size_t)b * p.T + t) : ((2u << t) - 1u)) : 0u;
#pragma unroll 1
          for (int r = 0; r < CW; ++r) {
            if (!valid || (rel >= 0 && !((msk >> (rel & 31)) & 1u))) dead |= 1ull << r;
            if (++hh == p.g) {
              hh = 0;
              ++t;
              if (t < p.T) msk = p.tree_mask ? __ldg(p.tree_mask + (size_t)b * p.T + t) : ((2u << t) - 1u);
            }
          }
        }
        twait(&sfull[sb], (tt >> 1) & 1, nullptr);
        fence_after();
        // pass 1: does any score exceed its row maximum by > 2^8 (or meet m = -inf)?  Outside a
        // unit's edge stage nothing is masked: padded rows (r >= R, zero queries) are computed like
        // live ones there -- harmless, their outputs are never stored -- so the common stage has no
        // per-element tests (E = false)
        auto pass1 = [&](auto edge_c) -> float {
          constexpr bool E = decltype(edge_c)::value;
          float xm = -INFINITY;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            float v[CH];
            tload(s_col + ch * CH, v);
#pragma unroll
            for (int r = 0; r < CH; r += 4) {
              const float4 m4 = *reinterpret_cast<const float4*>(mrow + cb + ch * CH + r);
              const float mm[4] = {m4.x, m4.y, m4.z, m4.w};
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                const float xv = fmaf(v[r + i], sl2, -mm[i]);
                xm = fmaxf(xm, (E && ((dead >> (ch * CH + r + i)) & 1ull)) ? -INFINITY : xv);
              }
            }
          }
          return xm;
        };
        const float xmax = edge ? pass1(std::true_type()) : pass1(std::false_type());
        if (tt > 0) twait(pempty, (tt - 1) & 1, nullptr);  // previous PV done: P and O^T are free
        if (vote_any128(xmax > THR, bar_id)) {
          // raise the group's row maxima to this tile's: per-row max over the 128 keys
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            float v[CH];
            tload(s_col + ch * CH, v);
#pragma unroll
            for (int i = 0; i < CH; ++i) {
              const int r = ch * CH + i;
              float m = (edge && ((dead >> r) & 1ull)) ? -INFINITY : v[i] * sl2;
#pragma unroll
              for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
              if (lane == 0) gred[wq * CW + r] = m;
            }
          }
          bar128(bar_id);
          if (x < CW) {
            const float m = fmaxf(fmaxf(gred[x], gred[CW + x]), fmaxf(gred[2 * CW + x], gred[3 * CW + x]));
            const float mo = mrow[cb + x];
            const float mn = fmaxf(mo, m);
            crow[cb + x] = (mo == -INFINITY) ? 0.f : ex2(mo - mn);
            mrow[cb + x] = mn;
          }
          bar128(bar_id);
#pragma unroll
          for (int r = 0; r < CW; ++r) lacc[r] *= crow[cb + r];
          if (j > 0) {  // O^T already holds PV of earlier tiles of this segment: rescale it
            const uint32_t oa = tbase + 2 * NP + ob * NP + cb + lane_off;
#pragma unroll
            for (int c = 0; c < CW; c += 16) {
              float o[16];
              tld16(oa + c, o);
              wait_ld();
#pragma unroll
              for (int i = 0; i < 16; ++i) o[i] *= (cb + c + i < R) ? crow[cb + c + i] : 0.f;
              tst16(oa + c, o);
            }
            wait_st();
          }
        }
        // pass 2: P = 2^(s * scale * log2 e - m) for the group's rows; row sums in fp32, the MMA
        // operand is bf16 (P^T core layout: key x -> core column x / 8, row (x % 8) * 16 B)
        uint8_t* pd = pbuf + (x >> 3) * 128 + (x & 7) * 16 + (cb / 8) * 2048;
        auto pass2 = [&](auto edge_c) {
          constexpr bool E = decltype(edge_c)::value;
#pragma unroll
          for (int ch = 0; ch < NCH; ++ch) {
            float v[CH];
            tload(s_col + ch * CH, v);
            uint32_t pk[CH / 2];
#pragma unroll
            for (int r = 0; r < CH; r += 4) {
              const float4 m4 = *reinterpret_cast<const float4*>(mrow + cb + ch * CH + r);
              const float mm[4] = {m4.x, m4.y, m4.z, m4.w};
              float pr[4];
#pragma unroll
              for (int i = 0; i < 4; ++i) {
                pr[i] = (E && ((dead >> (ch * CH + r + i)) & 1ull)) ? 0.f : ex2(fmaf(v[r + i], sl2, -mm[i]));
                lacc[ch * CH + r + i] += pr[i];
              }
              pk[r / 2] = pack_bf16(pr[0], pr[1]);
              pk[r / 2 + 1] = pack_bf16(pr[2], pr[3]);
            }
#pragma unroll
            for (int c = 0; c < CH / 8; ++c)
              *reinterpret_cast<uint4*>(pd + (ch * CH / 8 + c) * 2048) =
                  make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
          }
        };
        if (edge) pass2(std::true_type());
        else pass2(std::false_type());
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[sb]);  // S^T buffer sb is read for the last time
        if (!valid && grp == 0) {  // zero this key's V row once (after the V half's TMA writes land)
          mbar_wait(&vfull[stage], (it / NSTAGE) & 1);
          zero_vrow(ring + stage * STAGE + 2 * SLAB + x * 128, x);
        }
        fence_proxy_async();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(pfull);
      }
      // ---------------- segment epilogue: the group's row sums, O^T / l
#pragma unroll
      for (int r = 0; r < CW; ++r) {
        float l = lacc[r];
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
        if (lane == 0) gred[wq * CW + r] = l;
      }
      bar128(bar_id);
      if (x < CW) crow[cb + x] = gred[x] + gred[CW + x] + gred[2 * CW + x] + gred[3 * CW + x];  // L_r
      bar128(bar_id);
      mbar_wait(&ofull[ob], (si >> 1) & 1);
      fence_after();
      const bool complete = sg.complete();
      const int slot_base = seg_slot(p, pl, sg, chunk);
#pragma unroll
      for (int ch = 0; ch < NCH; ++ch) {
        float o[CH];
        tload(tbase + 2 * NP + ob * NP + cb + ch * CH + lane_off, o);
#pragma unroll
        for (int i = 0; i < CH; ++i) {
          const int row = cb + ch * CH + i;
          if (row < R) {
            const float L = crow[row];
            const float val = (L > 0.f) ? o[i] / L : 0.f;
            if (complete) store_out(p, o_row(p, b, kvh, row) * D + x, val);
            else __stcg(p.ws_o + ((int64_t)slot_base * p.R + row) * D + x, val);
          }
        }
      }
      fence_before();
      __syncwarp();
      if (lane == 0) mbar_arrive(&oempty[ob]);
      if (x < CW && cb + x < R) {
        const float L = crow[cb + x], m = mrow[cb + x];
        const float lse2 = (L > 0.f) ? m + __log2f(L) : -INFINITY;
        if (complete) {
          if (p.lse != nullptr) p.lse[out_row(p, b, kvh, cb + x)] = lse2 * LN2;
        } else {
          __stcg(p.ws_lse + (int64_t)slot_base * p.R + cb + x, lse2);
        }
      }
      if (!complete) finish_unit<D>(p, sg, pl, SM_THREADS, flag);
      bar128(bar_id);  // the group's red / mrow / crow entries are reused by the next segment
      ++si;
    }
  }
  fence_before();
  __syncthreads();
  if (!p.pdl_early) pdl_trigger();
  if (warp == ISSUER) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::TMEM_COLS));
  }
}

}  // namespace tc
