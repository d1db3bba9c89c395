// attn_exp_fma.cuh — EXPERIMENT ONLY (A/B builds with -DMD_EXP_FMA=1, tools/build_variant.py):
// the draft segment of attn_keys_kernel on CUDA-core FMA instead of mma.sync.  Included by
// attn.cu only under MD_EXP_FMA; the product library never compiles it.  Measured 1.35x slower
// (profiles/draft_ab_r02_fma_l2pf.txt), kept so the A/B can be re-run.
#pragma once

// EXPERIMENT (A/B builds only, -DMD_EXP_FMA=1): the draft segment on CUDA-core FMA instead of
// mma.sync, as north_star's "otherwise CUDA-core FMA" reads for R = g <= 4 query rows.  Same
// producer, ring, stage protocol and cross-CTA finish; consumer warp w takes keys 16w..16w+15 of
// each tile.  S: lane (half = lane/16, key = lane%16) dots its key's K half-row (64 d, LDS.128
// from the swizzled tile) with the segment's Q converted once to fp32 in shared memory, the two
// halves meet by one shuffle; the row max by 4 shuffles.  PV: lane owns d = 4 lane .. 4 lane + 3,
// reads P[key][0..3] as one broadcast LDS.128 and V[key][its 4 d] as one LDS.64, 16 FFMA per key.
// Epilogue: every warp parks its scaled [4][D] rows in the epilogue buffer, the CTA sums them.
MD_DEV uint4 lds128(uint32_t a) {
  uint4 v;
  asm volatile("ld.shared.v4.u32 {%0, %1, %2, %3}, [%4];" : "=r"(v.x), "=r"(v.y), "=r"(v.z), "=r"(v.w) : "r"(a));
  return v;
}
MD_DEV uint2 lds64(uint32_t a) {
  uint2 v;
  asm volatile("ld.shared.v2.u32 {%0, %1}, [%2];" : "=r"(v.x), "=r"(v.y) : "r"(a));
  return v;
}
MD_DEV float bf_lo(uint32_t x) { return __uint_as_float(x << 16); }
MD_DEV float bf_hi(uint32_t x) { return __uint_as_float(x & 0xffff0000u); }

template <int D, typename C>
__device__ void fma_segment(const AttnParams& p, const Plan& pl, const Seg& sg, int chunk, uint32_t ring, uint8_t* qbuf,
                            float* obuf, float* mlbuf, float* lsebuf, uint64_t* full, uint64_t* empty, uint64_t* qfull,
                            uint64_t* qempty, int* flag, int& it, int& qi) {
  constexpr int RF = 4, NC = C::NC, NSTAGE = C::NSTAGE, KS = C::NC;
  static_assert(C::KW == 16, "one 16-key slice per consumer warp");
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const Ranges rg = seg_ranges(p, sg);
  float* qf = obuf;                              // [RF][D] fp32 Q of this segment
  float* pw = obuf + RF * D + warp * 16 * RF;    // this warp's P [16 keys][RF]
  {
    const int qs = qi & 1;
    mbar_wait(&qfull[qs], (qi >> 1) & 1);
    for (int i = threadIdx.x; i < RF * D; i += NC * 32) {
      const int r = i / D, c = i - r * D;
      const uint16_t* qrow = reinterpret_cast<const uint16_t*>(qbuf + (qs * C::ROWS + r) * C::QSTR);
      qf[i] = __uint_as_float((uint32_t)qrow[c] << 16);  // rows >= R are zero
    }
    named_bar_sync(1, NC * 32);
    if (lane == 0) mbar_arrive(&qempty[qs]);
    ++qi;
  }
  const uint32_t qfa = smem_u32(qf), pwa = smem_u32(pw);
  const int half = lane >> 4, kl = lane & 15, ch = lane >> 1;
  float o[RF][4], m[RF], l[RF];
#pragma unroll
  for (int r = 0; r < RF; ++r) {
    o[r][0] = o[r][1] = o[r][2] = o[r][3] = 0.f;
    m[r] = -INFINITY;
    l[r] = 0.f;
  }
#pragma unroll 1
  for (int part = 0; part < 2; ++part) {
    const int rs = part ? rg.s1 : rg.s0, re = part ? rg.e1 : rg.e0;
#pragma unroll 1
    for (int pos = rs; pos < re; pos += TK, ++it) {
      const int stage = it % NSTAGE;
      mbar_wait(&full[stage], (it / NSTAGE) & 1);
      const int nvalid = min(TK, re - pos);
      const int kw0 = warp * 16;
      if (kw0 < nvalid) {
        const uint32_t kt = ring + stage * C::STAGE, vt = kt + C::TILE;
        const int key = kw0 + kl;
        float s[RF] = {0.f, 0.f, 0.f, 0.f};
#pragma unroll
        for (int c = 0; c < 8; ++c) {
          const uint4 kv = lds128(kt + half * (TK * 128) + swz128(key, c));
          const float kf[8] = {bf_lo(kv.x), bf_hi(kv.x), bf_lo(kv.y), bf_hi(kv.y),
                               bf_lo(kv.z), bf_hi(kv.z), bf_lo(kv.w), bf_hi(kv.w)};
#pragma unroll
          for (int r = 0; r < RF; ++r) {
            const uint32_t qa = qfa + (uint32_t)((r * D + half * 64 + c * 8) * 4);
            const uint4 q0 = lds128(qa), q1 = lds128(qa + 16);
            float a = s[r];
            a = fmaf(__uint_as_float(q0.x), kf[0], a);
            a = fmaf(__uint_as_float(q0.y), kf[1], a);
            a = fmaf(__uint_as_float(q0.z), kf[2], a);
            a = fmaf(__uint_as_float(q0.w), kf[3], a);
            a = fmaf(__uint_as_float(q1.x), kf[4], a);
            a = fmaf(__uint_as_float(q1.y), kf[5], a);
            a = fmaf(__uint_as_float(q1.z), kf[6], a);
            a = fmaf(__uint_as_float(q1.w), kf[7], a);
            s[r] = a;
          }
        }
        const bool valid = key < nvalid;
        float mx[RF];
#pragma unroll
        for (int r = 0; r < RF; ++r) {
          s[r] += __shfl_xor_sync(0xffffffffu, s[r], 16);
          s[r] = valid ? s[r] * p.scale_log2 : -INFINITY;
          mx[r] = s[r];
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 1));
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 2));
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 4));
          mx[r] = fmaxf(mx[r], __shfl_xor_sync(0xffffffffu, mx[r], 8));
        }
        bool moved = false;
        float corr[RF];
#pragma unroll
        for (int r = 0; r < RF; ++r) {
          const float mn = fmaxf(m[r], mx[r]);
          const float base = (mn == -INFINITY) ? 0.f : mn;
          corr[r] = ex2(m[r] - base);
          moved |= corr[r] != 1.f;
          m[r] = mn;
          s[r] = ex2(s[r] - base);
          l[r] = l[r] * corr[r] + (half == 0 ? s[r] : 0.f);
        }
        if (moved) {  // warp-uniform: m, mx are identical in every lane
#pragma unroll
          for (int r = 0; r < RF; ++r)
#pragma unroll
            for (int j = 0; j < 4; ++j) o[r][j] *= corr[r];
        }
        if (half == 0) *reinterpret_cast<float4*>(pw + kl * RF) = make_float4(s[0], s[1], s[2], s[3]);
        __syncwarp();
        const int kmax = min(16, nvalid - kw0);
        const uint32_t vb = vt + (ch >> 3) * (TK * 128) + (lane & 1) * 8;
#pragma unroll
        for (int k = 0; k < 16; ++k) {
          if (k >= kmax) break;  // rows past the valid keys may hold non-finite bits: never read
          const uint4 pp = lds128(pwa + k * RF * 4);
          const uint2 vv = lds64(vb + swz128(kw0 + k, ch & 7));
          const float v[4] = {bf_lo(vv.x), bf_hi(vv.x), bf_lo(vv.y), bf_hi(vv.y)};
          const float pr[4] = {__uint_as_float(pp.x), __uint_as_float(pp.y), __uint_as_float(pp.z),
                               __uint_as_float(pp.w)};
#pragma unroll
          for (int r = 0; r < RF; ++r)
#pragma unroll
            for (int j = 0; j < 4; ++j) o[r][j] = fmaf(pr[r], v[j], o[r][j]);
        }
        __syncwarp();
      }
      __syncwarp();
      if (lane == 0) mbar_arrive(&empty[stage]);
    }
  }
  // ------------------------------------------------------------ epilogue
#pragma unroll
  for (int r = 0; r < RF; ++r) {
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 1);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 2);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 4);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 8);
    l[r] += __shfl_xor_sync(0xffffffffu, l[r], 16);  // lanes 16..31 hold 0: every lane gets the total
  }
  if (lane == 0) {
#pragma unroll
    for (int r = 0; r < RF; ++r) {
      mlbuf[(warp * C::ROWS + r) * 2 + 0] = m[r];
      mlbuf[(warp * C::ROWS + r) * 2 + 1] = l[r];
    }
  }
  named_bar_sync(1, NC * 32);  // every warp is past its tile loop: qf / pw may be overwritten
#pragma unroll
  for (int r = 0; r < RF; ++r) {
    float M = -INFINITY, L = 0.f;
#pragma unroll
    for (int k = 0; k < KS; ++k) M = fmaxf(M, mlbuf[(k * C::ROWS + r) * 2]);
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      const float* e = &mlbuf[(k * C::ROWS + r) * 2];
      if (e[1] > 0.f) L += e[1] * ex2(e[0] - M);
    }
    const float f = (l[r] > 0.f) ? ex2(m[r] - M) / L : 0.f;
    if (warp == 0 && lane == 0) lsebuf[r] = (L > 0.f) ? M + __log2f(L) : -INFINITY;
    *reinterpret_cast<float4*>(obuf + (warp * RF + r) * D + lane * 4) =
        make_float4(o[r][0] * f, o[r][1] * f, o[r][2] * f, o[r][3] * f);
  }
  named_bar_sync(1, NC * 32);
  const bool complete = sg.complete();
  const int slot_base = seg_slot(p, pl, sg, chunk);
  constexpr int V4 = D / 4;
  for (int idx = threadIdx.x; idx < p.R * V4; idx += NC * 32) {
    const int r = idx / V4, c4 = (idx - r * V4) * 4;
    float4 v = make_float4(0.f, 0.f, 0.f, 0.f);
#pragma unroll
    for (int w = 0; w < NC; ++w) {
      const float4 a = *reinterpret_cast<const float4*>(obuf + (w * RF + r) * D + c4);
      v.x += a.x;
      v.y += a.y;
      v.z += a.z;
      v.w += a.w;
    }
    if (complete) {
      store_out(p, o_row(p, sg.b, sg.kvh, r) * D + c4, v);
      if (c4 == 0 && p.lse != nullptr) p.lse[out_row(p, sg.b, sg.kvh, r)] = lsebuf[r] * LN2;
    } else {
      const int64_t prow = (int64_t)slot_base * p.R + r;
      __stcg(reinterpret_cast<float4*>(p.ws_o + prow * D + c4), v);
      if (c4 == 0) __stcg(p.ws_lse + prow, lsebuf[r]);
    }
  }
  if (!complete) finish_unit<D>(p, sg, pl, NC * 32, flag);
  named_bar_sync(1, NC * 32);  // the epilogue buffers are reused by the next segment
}
