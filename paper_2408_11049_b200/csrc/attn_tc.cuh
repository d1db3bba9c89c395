// attn_tc.cuh — the tcgen05 (5th-generation tensor core) verify kernel, included by attn.cu
// after the stream-K machinery (AttnParams, Plan, SegWalker, finish_unit) it reuses.
//
// md_verify_attn_full for R = g*(gamma+1) in (8, 48] query rows per KV head at head_dim 128
// (GQA verify: Llama-3.1 R = 20, Qwen2.5 R = 35).  Swapped operands so
// the tensor-core work is 2 * 128 * NP FLOP per key (NP = R rounded up to 16), not 128 rows:
//   S^T[128 keys][NP]  = K[128 keys][d] . Q^T            (A = K tile, K-major SW128 from TMA;
//                                                          B = Q rows, K-major SW128 from TMA)
//   O^T[d][NP]        += V^T . P^T                       (A = V tile read MN-major, SW128;
//                                                          B = P^T, MN-major 8x8 core matrices)
// Both accumulators live in TMEM (S^T double-buffered by tile, O^T by segment).  Warp roles
// (192 threads, 1 CTA / SM, 3 x 64 KB K/V stages of 128 keys):
//   warp 4  TMA producer: the segment's Q rows (one 3-D box per 64-column slab) and K/V tiles;
//   warp 5  MMA issuer (one thread) + TMEM allocator: S^T(i) is issued before PV(i-1);
//   warps 0-3 softmax + epilogue, thread x <-> TMEM lane x (key x of the tile for S^T, head
//           dim x for O^T): each thread owns one key's NP scores, so the online softmax needs
//           no cross-thread work per tile except a CTA vote: the running row maxima m are only
//           raised when a score exceeds m + 8 (log2 units; P stays <= 2^8, exact in the
//           fp32 sums and a bf16 operand like any other), which rescales the thread-local row
//           sums and O^T in TMEM (tcgen05.ld/st); row sums are reduced across the 128 threads
//           once per segment.  Keys past the tile's valid range get P = 0 and their V rows
//           are zeroed in shared memory (fetched cache rows past kv_len may hold NaN bits).
// Stream-K decomposition, split partials and the fused last-arriver merge are those of the
// mma.sync kernels (64-key plan tiles; a 128-key stage covers two of them).

namespace tc {  // helpers: tcgen05.cuh (included by attn.cu)

constexpr int KT = 128;                      // keys per stage (MMA M)
constexpr int SLAB = KT * 128;               // one 64-column slab of a 128-key tile
constexpr int STAGE = 4 * SLAB;              // K (2 slabs) + V (2 slabs) = 64 KB
constexpr float THR = 8.f;                   // lazy max-raise threshold (log2 units)
constexpr int SM_THREADS = 128;              // softmax / epilogue threads
constexpr int THREADS = SM_THREADS + 64;     // + producer warp + MMA warp

template <int NP>
struct Cfg {
  static constexpr int NQ = NP <= 32 ? 2 : 1;        // Q buffers (by segment parity)
  static constexpr int QBUF = 2 * NP * 128;          // Q rows, two 64-column SW128 slabs
  static constexpr int PBUF = NP * KT * 2;           // P^T, 8x8 core matrices
  static constexpr int NSTAGE = 3;
  static constexpr int AUX = 2048 + TABLE_BYTES;     // barriers, tmem slot, row state, plan
  static constexpr int SMEM = NSTAGE * STAGE + NQ * QBUF + PBUF + AUX + 1024;
  static constexpr int TMEM_COLS = 4 * NP <= 128 ? 128 : 256;  // S^T x2 + O^T x2
  static_assert(SMEM <= 232448, "shared memory budget");
};

// OR-vote over the 128 softmax threads (named barrier 2)
__device__ __forceinline__ bool vote_any128(bool v) {
  uint32_t r;
  asm volatile(
      "{\n\t.reg .pred q, p;\n\tsetp.ne.u32 q, %1, 0;\n\tbarrier.cta.red.or.pred p, 2, 128, q;\n\t"
      "selp.u32 %0, 1, 0, p;\n\t}"
      : "=r"(r)
      : "r"((uint32_t)v)
      : "memory");
  return r != 0;
}
__device__ __forceinline__ void bar128() { named_bar_sync(2, SM_THREADS); }

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

// RR > 0: the row count R is a compile-time constant (the hot configurations), else p.R
template <int NP, int RR>
__global__ void __launch_bounds__(THREADS, 1)
    attn_tc_kernel(const __grid_constant__ TmapSet tm, const __grid_constant__ CUtensorMap qmap, const AttnParams p) {
  using C = Cfg<NP>;
  const int R = RR > 0 ? RR : p.R;
  constexpr int NSTAGE = C::NSTAGE, NQ = C::NQ;
  constexpr int D = 128;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* smem = smem_raw + ((1024u - (smem_u32(smem_raw) & 1023u)) & 1023u);
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
  uint64_t* cfull = oempty + 2;      // [2] dynamic chunk hand-off, producer -> MMA + softmax
  uint64_t* cempty = cfull + 2;      // [2]
  uint64_t* vfull = cempty + 2;      // [NSTAGE] V halves of the ring stages (full / empty: K halves)
  uint64_t* vempty = vfull + NSTAGE; // [NSTAGE]
  uint64_t* apb = vempty + NSTAGE;   // [1] fused append: the softmax warps' new-row stores are done
  int* cids = reinterpret_cast<int*>(apb + 1);  // [2]
  uint32_t* tslot = reinterpret_cast<uint32_t*>(cids + 2);
  int* flag = reinterpret_cast<int*>(tslot + 4);                 // [16] finish_unit
  Plan* plan_smem = reinterpret_cast<Plan*>(flag + 16);          // 40 bytes (reserved 64)
  float* red = reinterpret_cast<float*>(flag + 32);              // [4][NP] per-warp row maxima / sums
  float* mrow = red + 4 * NP;                                    // [NP] running row maxima (log2 units)
  float* crow = mrow + NP;                                       // [NP] rescale factors
  int* pre = reinterpret_cast<int*>(crow + NP);                  // [TABLE_B + 1]

  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
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
      mbar_init(&sempty[s], 4);
      mbar_init(&ofull[s], 1);
      mbar_init(&oempty[s], 4);
    }
    mbar_init(pfull, 4);
    mbar_init(pempty, 1);
    for (int s2 = 0; s2 < 2; ++s2) {
      mbar_init(&cfull[s2], 1);
      mbar_init(&cempty[s2], 5);  // the MMA thread + one arrival per softmax warp
    }
    mbar_init(apb, 4);
    fence_mbar_init();
  }
  // Q rows >= R stay zero for the whole kernel (the TMA boxes write rows < R only)
  for (int i = threadIdx.x; i < NQ * C::QBUF / 16; i += THREADS) {
    const int slab_row = (i * 16 / 128) % NP;
    if (slab_row >= p.R) reinterpret_cast<uint4*>(qbuf)[i] = make_uint4(0, 0, 0, 0);
  }
  fence_proxy_async();
  if (warp == 5) {
    asm volatile("tcgen05.alloc.cta_group::1.sync.aligned.shared::cta.b32 [%0], %1;" ::"r"(smem_u32(tslot)),
                 "n"(C::TMEM_COLS));
    asm volatile("tcgen05.relinquish_alloc_permit.cta_group::1.sync.aligned;");
  }
  if (warp == 4 && lane == 0) {  // descriptor fetches overlap the grid-dependency wait
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
  const Plan& pl = *plan_smem;
  int chunk = blockIdx.x;  // this CTA's static chunk, then the dynamic ones its producer claims
  const bool active = (int)blockIdx.x < pl.G;
  SegWalker walk;
  Seg sg;
  if (active) walk.init(p, pre, pl.start(chunk), pl.start(chunk + 1));
  if (p.kn != nullptr && warp < 4 && active) {  // fused append: the new rows of this CTA's tiles
    append_own_rows<128>(p, pre, pl.start(chunk), pl.start(chunk + 1), threadIdx.x, SM_THREADS);
    __syncwarp();
    if (lane == 0) mbar_arrive(apb);
  }

  if (warp == 4) {
    // ============================== TMA producer ==============================
    if (active && lane == 0) {
      prefetch_tmap(&tm.k_full);
      prefetch_tmap(&tm.v_full);
      prefetch_tmap(&tm.k_part);
      prefetch_tmap(&tm.v_part);
      prefetch_tmap(&qmap);
      const uint64_t pol = policy_evict_first();
      int it = 0, qi = 0, ck = 0;
      PendV pend{-1, 0, 0, 0, 0};
      long long tw = 0;
      long long* twp = p.trace ? &tw : nullptr;
      // dynamic tail (long calls, see make_plan): chunks claimed one ahead from an atomic
      // counter and handed to the MMA and softmax roles through a 2-slot mbarrier ring
      int ahead = 0;
      if (pl.nch > pl.G) ahead = atomicAdd(p.dyn, 1);
      while (true) {
        if (!walk.next(p, pre, sg)) {
          if (pl.nch == pl.G) break;
          const int c = pl.G + ahead;
          const int nxt = c < pl.nch ? c : -1;
          if (nxt >= 0) ahead = atomicAdd(p.dyn, 1);
          const int cs = ck & 1;
          mbar_wait(&cempty[cs], ((ck >> 1) & 1) ^ 1);
          cids[cs] = nxt;
          mbar_arrive(&cfull[cs]);
          ++ck;
          if (nxt < 0) break;
          chunk = nxt;
          walk.init(p, pre, pl.start(chunk), pl.start(chunk + 1));
          continue;
        }
        produce<NP>(p, tm, &qmap, sg, seg_ranges(p, sg), ring, qbuf, full, empty, vfull, vempty, qfull, qempty, it, qi,
                    pend, pol, twp, apb);
      }
      if (pend.it >= 0) issue_v<NSTAGE>(tm, ring, vfull, vempty, pend, pol);
      if (p.trace) trace_put(p, 15, tw);
    }
  } else if (warp == 5) {
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
      int pv_stage = -1, pv_ob = 0, pv_first = 0, pv_last = 0, pv_qs = 0, pv_tt = 0, pv_it = 0;
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
      int ck = 0;
      auto next_seg = [&]() -> bool {  // mirrors the producer's chunk sequence
        while (!walk.next(p, pre, sg)) {
          if (pl.nch == pl.G) return false;
          const int cs = ck & 1;
          mbar_wait(&cfull[cs], (ck >> 1) & 1);
          const int nxt = cids[cs];
          mbar_arrive(&cempty[cs]);
          ++ck;
          if (nxt < 0) return false;
          chunk = nxt;
          walk.init(p, pre, pl.start(chunk), pl.start(chunk + 1));
        }
        return true;
      };
      while (next_seg()) {
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
          pv_qs = qs;
          pv_tt = tt;
          pv_it = it;
        }
        ++qi;
        ++si;
      }
      if (pv_stage >= 0) issue_pv();
      (void)pv_qs;
      if (p.trace) {
        trace_put(p, 8, w_full);
        trace_put(p, 9, w_se);
        trace_put(p, 10, w_pf);
        trace_put(p, 11, tt);
      }
    }
  } else if (active) {
    // ============================== softmax + epilogue (128 threads) ==============================
    const int x = threadIdx.x;                      // TMEM lane: key of the tile / head-dim row of O^T
    const uint32_t lane_off = (uint32_t)(warp * 32) << 16;
    int it = 0, tt = 0, si = 0;
    long long w_sf = 0, w_pe = 0, w_epi = 0, t_start = clock64();
    long long* wsf = (p.trace && x == 0) ? &w_sf : nullptr;
    long long* wpe = (p.trace && x == 0) ? &w_pe : nullptr;
    long long sec[6] = {0, 0, 0, 0, 0, 0}, tsec = 0;
    const bool prof = p.trace && x == 0;
#define TSEC(k)                              \
  if (prof) {                                \
    const long long tn = clock64();          \
    sec[k] += tn - tsec;                     \
    tsec = tn;                               \
  }
    float mr[NP], lacc[NP];
    int ck = 0;
    auto next_seg = [&]() -> bool {  // mirrors the producer's chunk sequence
      while (!walk.next(p, pre, sg)) {
        if (pl.nch == pl.G) return false;
        const int cs = ck & 1;
        mbar_wait(&cfull[cs], (ck >> 1) & 1);
        const int nxt = cids[cs];
        __syncwarp();
        if (lane == 0) mbar_arrive(&cempty[cs]);
        ++ck;
        if (nxt < 0) return false;
        chunk = nxt;
        walk.init(p, pre, pl.start(chunk), pl.start(chunk + 1));
      }
      return true;
    };
    while (next_seg()) {
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
        if (prof) tsec = clock64();
        fence_after();
        float v[NP];
#pragma unroll
        for (int c = 0; c < NP; c += 16) tld16(tbase + sb * NP + c + lane_off, v + c);
        wait_ld();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(&sempty[sb]);
        TSEC(0)
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
        TSEC(1)
        // the previous tile's PV must be complete before P is rewritten or O^T rescaled
        if (tt > 0) twait(pempty, (tt - 1) & 1, wpe);
        if (prof) tsec = clock64();
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
        TSEC(2)
        // P = 2^x; row sums accumulate in fp32, the MMA operand is bf16
        uint32_t pk[NP / 2];
#pragma unroll
        for (int r = 0; r < NP; r += 2) {
          const float p0 = (r < R) ? ex2(xs[r]) : 0.f, p1 = (r + 1 < R) ? ex2(xs[r + 1]) : 0.f;
          lacc[r] += p0;
          lacc[r + 1] += p1;
          pk[r / 2] = pack_bf16(p0, p1);
        }
        TSEC(3)
        // P^T core layout: key x -> core column x / 8, row (x % 8) * 16 B; rows r -> core r / 8
        uint8_t* pd = pbuf + (x >> 3) * 128 + (x & 7) * 16;
#pragma unroll
        for (int c = 0; c < NP / 8; ++c)
          *reinterpret_cast<uint4*>(pd + c * 2048) = make_uint4(pk[4 * c], pk[4 * c + 1], pk[4 * c + 2], pk[4 * c + 3]);
        if (!valid) {  // zero this key's V row (cache rows past the valid keys may hold NaN bits)
          mbar_wait(&vfull[stage], (it / NSTAGE) & 1);  // after the V half's TMA writes land
          uint8_t* vrow = ring + stage * STAGE + 2 * SLAB + x * 128;
#pragma unroll
          for (int c = 0; c < 8; ++c) {
            *reinterpret_cast<uint4*>(vrow + c * 16) = make_uint4(0, 0, 0, 0);
            *reinterpret_cast<uint4*>(vrow + SLAB + c * 16) = make_uint4(0, 0, 0, 0);
          }
        }
        TSEC(4)
        fence_proxy_async();
        fence_before();
        __syncwarp();
        if (lane == 0) mbar_arrive(pfull);
        TSEC(5)
      }
      // ---------------- segment epilogue: row sums over the 128 key lanes, O^T / l
      const long long t_epi = prof ? clock64() : 0;
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
      const int slot_base = chunk * 2 + pl.slot(sg.ustart, chunk);
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
      if (!complete && p.fused_merge) finish_unit<D>(p, sg, pl, SM_THREADS, flag);
      bar128();  // red / mrow / crow reused by the next segment
      if (prof) w_epi += clock64() - t_epi;
      ++si;
    }
    if (p.trace && x == 0) {
      trace_put(p, 12, w_sf);
      trace_put(p, 13, w_pe);
      trace_put(p, 14, clock64() - t_start);
      trace_put(p, 7, w_epi);  // segment epilogues (row sums, O^T read, stores, split merge)
      trace_put(p, 6, globaltimer());  // softmax end (ns): the CTA's finish time
      for (int k = 0; k < 6; ++k) trace_put(p, k, sec[k]);
    }
#undef TSEC
  }
  // the last CTA to finish re-arms the dynamic counters for the next call (every producer has
  // made its final claim before any role saw the -1 hand-off)
  if (active && pl.nch > pl.G && threadIdx.x == 0) {
    if (atomicAdd(p.dyn + 1, 1) == pl.G - 1) {
      p.dyn[0] = 0;
      p.dyn[1] = 0;
    }
  }
  fence_before();
  __syncthreads();
  if (!p.pdl_early) pdl_trigger();
  if (warp == 5) {
    fence_after();
    asm volatile("tcgen05.dealloc.cta_group::1.sync.aligned.b32 %0, %1;" ::"r"(tbase), "n"(C::TMEM_COLS));
  }
}

}  // namespace tc
