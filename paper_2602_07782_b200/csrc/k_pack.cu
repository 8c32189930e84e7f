// k_pack.cu -- K4: balanced fold-and-push for every candidate scale in ONE
// launch (one CTA per candidate, "one work group per scale factor"),
// and K5: scale selection + placement scatter.
//
// Per candidate the CTA runs Alg. 4 row by row with the frontline
// F (one int32 per dilated atlas column) resident in shared memory:
//   Alg. 2 knee refinement (block arg-max/min over F)
//   Alg. 3 fold of both HC settings as two block-wide exclusive
//   scans + first-overflow min-reductions
//   non-adjacent lock pairs of the row (D15)
//   push: warp per (config, chart), max over covered columns of
//   F - TopEdge (reads the packed footprints, coalesced)
//   Alg. 1 fixpoint over the lock pairs
//   score: max over covered columns of Y + BottomEdge, per config
//   hierarchical selection, commit (shared atomicMax into F),
//   FindKnee (block max of the height drop)
// Selection is decided before pushing where the paper allows it: the
// horizontal-compaction choice depends only on the fold's row end (P:304
// "enable horizontal compacting if it allows more charts to fit"), so each
// fold pushes 2 directions instead of 4 configurations, with identical
// results.
#include "tabi_internal.cuh"

namespace tabi {
namespace {

constexpr int kNT = 512;
constexpr int kNW = kNT / 32;

struct Smem {
  int32_t scan[2][kNW + 1];
  int32_t row_start, fmax, fail, rows, knees_found, knee_rows;
  int32_t knee_valid, knee_ltr, knee_left, knee_right;
  int32_t nk, conc_max;
  int32_t endv[4];      // (fold f, hc) -> row end, index f * 2 + hc
  int32_t fmin[4];
  int32_t done;
  int32_t hcsel[2], knee_ok, end_cfg[4];
  int32_t newmax[4];
  int32_t changed, npairs, pair_overflow;
  int32_t sel_cfg;
  unsigned long long knee_key;
  unsigned long long work;
};

__device__ __forceinline__ void block_scan2(int32_t a, int32_t b, int32_t& ea, int32_t& eb,
                                            int32_t& ta, int32_t& tb, Smem& S) {
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int32_t ia = warp_incl_sum(a, lane), ib = warp_incl_sum(b, lane);
  if (lane == 31) { S.scan[0][wid] = ia; S.scan[1][wid] = ib; }
  __syncthreads();
  if (wid == 0) {
    const int32_t va = lane < kNW ? S.scan[0][lane] : 0, vb = lane < kNW ? S.scan[1][lane] : 0;
    const int32_t xa = warp_incl_sum(va, lane), xb = warp_incl_sum(vb, lane);
    if (lane < kNW) { S.scan[0][lane] = xa - va; S.scan[1][lane] = xb - vb; }
    if (lane == 31) { S.scan[0][kNW] = xa; S.scan[1][kNW] = xb; }
  }
  __syncthreads();
  ea = S.scan[0][wid] + ia - a;
  eb = S.scan[1][wid] + ib - b;
  ta = S.scan[0][kNW];
  tb = S.scan[1][kNW];
  __syncthreads();
}

__global__ void __launch_bounds__(kNT, 1)
pack_kernel(PackParams pp, const int32_t* __restrict__ colofs, const int32_t* __restrict__ rowofs,
            const uint32_t* __restrict__ dcol, const uint32_t* __restrict__ drow,
            const int32_t* __restrict__ wd_all, const int32_t* __restrict__ hd_all,
            const int32_t* __restrict__ off_all, const uint8_t* __restrict__ lock_all,
            const int32_t* __restrict__ hsorted, const int32_t* __restrict__ cand_bad,
            int32_t* scratch, int64_t pair_cap, int32_t* Xo_all, int32_t* Yo_all, uint8_t* mir_all,
            Cand* cands, Status* st) {
  extern __shared__ int32_t F[];
  __shared__ Smem S;
  const int tid = threadIdx.x, lane = tid & 31, wid = tid >> 5;
  const int m = blockIdx.x + 1;
  const int n = pp.n, Wp = pp.Wp, Hp = pp.Hp;
  if (st->bad_chart != INT32_MAX || st->capacity) return;
  const int64_t cb = (int64_t)(m - 1) * n;
  const int32_t* wd = wd_all + cb;
  const int32_t* hd = hd_all + cb;
  const int32_t* off = off_all + cb;
  const uint8_t* lk = lock_all + cb;
  const uint32_t* col = dcol + (int64_t)(m - 1) * pp.col_cap;
  const uint32_t* row = drow + (int64_t)(m - 1) * pp.row_cap;
  int32_t* sc = scratch + (int64_t)(m - 1) * (6 * (int64_t)n + 3 * pair_cap);
  int32_t* xs0 = sc;
  int32_t* xs1 = sc + n;
  int32_t* Yc = sc + 2 * (int64_t)n;  // [4][n]
  int32_t* pa = sc + 6 * (int64_t)n;
  int32_t* pb = pa + pair_cap;
  int32_t* plk = pb + pair_cap;
  int32_t* Xo = Xo_all + cb;
  int32_t* Yo = Yo_all + cb;
  uint8_t* mir = mir_all + cb;
  const bool adj_only = (pp.flags & TABI_F_ADJACENT_LOCKS_ONLY) != 0;
  const bool no_hc = (pp.flags & TABI_F_NO_HC) != 0;
  const bool no_bal = (pp.flags & TABI_F_NO_BALANCE) != 0;

  if (cand_bad[m - 1]) {  // some chart exceeds the dilated atlas at this scale
    if (tid == 0) cands[m - 1] = Cand{0, 0, 0, 0, 0, 0, 0, -1};
    return;
  }
  {  // work accounting: footprint entries K3 produced for this candidate
    unsigned long long pe = 0;
    for (int s = tid; s < n; s += kNT) pe += (unsigned long long)(wd[s] + hd[s]);
    for (int o = 16; o > 0; o >>= 1) pe += __shfl_xor_sync(0xffffffffu, pe, o);
    if (lane == 0) atomicAdd(&st->work_prof, pe);
  }
  for (int x = tid; x < Wp; x += kNT) F[x] = 0;  // frontline starts at the top
  if (tid == 0) {
    S.row_start = 0; S.fmax = 0; S.fail = 0; S.rows = 0; S.knees_found = 0; S.knee_rows = 0;
    S.knee_valid = 0; S.knee_ltr = 0; S.knee_left = 0; S.knee_right = 0;
    S.work = 0ull;
  }
  __syncthreads();

  while (true) {
    const int32_t rs = S.row_start;
    if (rs >= n || S.fail) break;
    // ---- Alg. 2 UpdateKneeLocation ---------------------------
    if (S.knee_valid) {
      const int32_t left = S.knee_left, right = S.knee_right, ltr = S.knee_ltr;
      const bool degenerate = ltr ? (right >= Wp) : (left <= 0);
      if (tid == 0) S.nk = ltr ? left - 1 : right;
      __syncthreads();
      if (!degenerate) {
        const int32_t ref = ltr ? F[right] : F[left - 1];
        for (int x = left + tid; x < right; x += kNT) {
          if (F[x] >= ref) {
            if (ltr) atomicMax(&S.nk, x);
            else atomicMin(&S.nk, x);
          }
        }
      }
      __syncthreads();
      if (tid == 0) {
        if (degenerate) {
          S.knee_valid = 0;
        } else if (ltr) {
          if (S.nk + 1 == left) S.knee_valid = 0;  // collapsed: discard (D20)
          else S.knee_right = S.nk + 1;
        } else {
          if (S.nk == right) S.knee_valid = 0;
          else S.knee_left = S.nk;
        }
        S.conc_max = INT32_MIN;
      }
      __syncthreads();
    }
    const int32_t kv = S.knee_valid;
    const int32_t ka = kv ? (S.knee_ltr ? S.knee_right : 0) : 0;   // knee fold region [ka, kb)
    const int32_t kb = kv ? (S.knee_ltr ? Wp : S.knee_left) : 0;
    if (kv) {
      int32_t mx = INT32_MIN;
      for (int x = ka + tid; x < kb; x += kNT) mx = max(mx, F[x]);
      mx = warp_max(mx);
      if (lane == 0) atomicMax(&S.conc_max, mx);
    }
    // ---- Alg. 3 FoldRow for both HC settings and both folds --------------
    if (tid < 4) { S.endv[tid] = INT32_MIN; }
    if (tid == 0) S.done = 0;
    __syncthreads();
    {
      int32_t carry0 = 0, carry1 = 0;
      for (int base = rs;; base += kNT) {
        if (tid < 4) S.fmin[tid] = INT32_MAX;
        const int s = base + tid;
        const bool valid = s < n;
        const int32_t w_s = valid ? wd[s] : 0;
        const int32_t a1 = valid ? off[s] : 0;
        int32_t e0, e1, t0, t1;
        block_scan2(w_s, a1, e0, e1, t0, t1, S);
        const int32_t x0 = carry0 + e0, x1 = carry1 + e1;
        if (valid) {
          xs0[s] = x0;
          xs1[s] = x1;
          if (x0 + w_s > Wp) atomicMin(&S.fmin[0], s);
          if (x1 + w_s > Wp) atomicMin(&S.fmin[1], s);
          if (x0 + w_s > kb - ka) atomicMin(&S.fmin[2], s);
          if (x1 + w_s > kb - ka) atomicMin(&S.fmin[3], s);
        }
        __syncthreads();
        if (tid == 0) {
          for (int q = 0; q < 4; q++)
            if (S.endv[q] == INT32_MIN && S.fmin[q] != INT32_MAX) S.endv[q] = S.fmin[q] - 1;
          if (S.endv[1] != INT32_MIN || base + kNT >= n) {
            for (int q = 0; q < 4; q++)
              if (S.endv[q] == INT32_MIN) S.endv[q] = n - 1;
            S.done = 1;
          }
        }
        __syncthreads();
        if (S.done) break;
        carry0 += t0;
        carry1 += t1;
      }
    }
    // ---- level 1 of the hierarchical choice: HC iff it fits more --
    if (tid == 0) {
      S.hcsel[0] = (!no_hc && S.endv[1] > S.endv[0]) ? 1 : 0;
      S.hcsel[1] = (!no_hc && S.endv[3] > S.endv[2]) ? 1 : 0;
      const int32_t ea = S.endv[S.hcsel[0]];
      const int32_t ek = S.endv[2 + S.hcsel[1]];
      S.knee_ok = kv && ek >= rs;
      S.end_cfg[0] = S.end_cfg[1] = ea;
      S.end_cfg[2] = S.end_cfg[3] = ek;
      if (ea < rs) S.fail = 1;  // first chart wider than the atlas (D22)
      for (int q = 0; q < 4; q++) S.newmax[q] = INT32_MIN;
      S.npairs = 0;
      S.pair_overflow = 0;
    }
    __syncthreads();
    if (S.fail) break;
    const int32_t knee_ok = S.knee_ok;
    const int32_t hc0 = S.hcsel[0], hc1 = S.hcsel[1];
    const int32_t endA = S.end_cfg[0], endK = S.end_cfg[2];
    const int32_t nA = endA - rs + 1, nK = knee_ok ? endK - rs + 1 : 0;
    // ---- D15: non-adjacent lock pairs of the row (HC folds only) ----------
    const int32_t R = max(hc0 ? endA : -1, (knee_ok && hc1) ? endK : -1);
    if (!adj_only && R > rs) {
      int32_t carry = 0;
      for (int base = rs; base <= R; base += kNT) {
        const int a = base + tid;
        int32_t cnt = 0;
        if (a <= R) {
          const int32_t xa = xs1[a], wa = wd[a];
          for (int b = a + 2; b <= R && xs1[b] - xa < wa; b++) cnt++;
        }
        int32_t ex, dummy, tot, tot2;
        block_scan2(cnt, 0, ex, dummy, tot, tot2, S);
        if (a <= R && cnt > 0) {
          int32_t p = carry + ex;
          const int32_t xa = xs1[a];
          for (int b = a + 2; b < a + 2 + cnt; b++, p++) {
            if (p < pair_cap) {
              pa[p] = a;
              pb[p] = b;
            }
          }
          (void)xa;
        }
        carry += tot;
      }
      if (tid == 0) {
        S.npairs = carry;
        if (carry > pair_cap) {
          S.pair_overflow = 1;
          atomicOr(&st->capacity, 2);
          atomicMax(&st->pad[0], carry);
        }
      }
      __syncthreads();
      if (S.pair_overflow) { if (tid == 0) S.fail = 1; __syncthreads(); break; }
      const int32_t np = S.npairs;
      for (int p = wid; p < np; p += kNW) {
        const int a = pa[p], b = pb[p];
        bool la, lb;
        warp_locks(row + rowofs[a], row + rowofs[b], hd[a], hd[b], xs1[b] - xs1[a], lane, la, lb);
        if (lane == 0) plk[p] = (la ? 1 : 0) | (lb ? 2 : 0);
      }
      __syncthreads();
    }
    const int32_t np = S.npairs;
    // ---- push: Y = max over covered columns of F - TopEdge ----
    const int32_t total = 2 * nA + 2 * nK;
    for (int it = wid; it < total; it += kNW) {
      int cfg, s;
      if (it < 2 * nA) { cfg = it / nA; s = rs + it % nA; }
      else { const int t = it - 2 * nA; cfg = 2 + t / nK; s = rs + t % nK; }
      const int f = cfg >> 1, dir = cfg & 1;
      const int hc = f ? hc1 : hc0;
      const int32_t a_f = f ? ka : 0, b_f = f ? kb : Wp;
      const int32_t W_s = wd[s];
      const int32_t xl = hc ? xs1[s] : xs0[s];
      const int32_t X = dir ? b_f - xl - W_s : a_f + xl;
      const uint32_t* cp = col + colofs[s];
      int32_t v = INT32_MIN;
      for (int i = lane; i < W_s; i += 32) {
        const int ii = dir ? W_s - 1 - i : i;
        v = max(v, F[X + i] - lo16(cp[ii]));
      }
      v = warp_max(v);
      if (lane == 0) {
        __stcg(&Yc[(int64_t)cfg * n + s], v);
        atomicAdd(&S.work, (unsigned long long)W_s);
      }
    }
    __syncthreads();
    // ---- Alg. 1 CorrectYOffsets over adjacent + non-adjacent pairs ---------
    {
      const int c0 = hc0 ? 0 : 2, c1 = (knee_ok && hc1) ? 4 : 2;  // hc1 configs [c0, c1)
      if (c1 > c0) {
        const int32_t per = (endA - rs) + (adj_only ? 0 : np);  // adjacent pairs + list
        while (true) {
          if (tid == 0) S.changed = 0;
          __syncthreads();
          for (int it = tid; it < (c1 - c0) * per; it += kNT) {
            const int cfg = c0 + it / per;
            const int q = it % per;
            const int32_t endc = S.end_cfg[cfg];
            int a, b, bits;
            if (q < endA - rs) {
              a = rs + q; b = a + 1;
              if (b > endc) continue;
              bits = lk[a];
            } else {
              const int p = q - (endA - rs);
              a = pa[p]; b = pb[p];
              if (b > endc) continue;
              bits = plk[p];
            }
            int32_t* Ya = &Yc[(int64_t)cfg * n + a];
            int32_t* Yb = &Yc[(int64_t)cfg * n + b];
            const int32_t ya = __ldcg(Ya), yb = __ldcg(Yb);
            if ((bits & 1) && ya < yb) { atomicMax(Ya, yb); S.changed = 1; }
            if ((bits & 2) && yb < ya) { atomicMax(Yb, ya); S.changed = 1; }
          }
          __syncthreads();
          if (!S.changed) break;
          __syncthreads();
        }
      }
    }
    // ---- score: max over covered columns of Y + BottomEdge ----
    for (int it = wid; it < total; it += kNW) {
      int cfg, s;
      if (it < 2 * nA) { cfg = it / nA; s = rs + it % nA; }
      else { const int t = it - 2 * nA; cfg = 2 + t / nK; s = rs + t % nK; }
      const int dir = cfg & 1;
      const int32_t W_s = wd[s];
      const uint32_t* cp = col + colofs[s];
      const int32_t y = __ldcg(&Yc[(int64_t)cfg * n + s]);
      int32_t v = INT32_MIN;
      for (int i = lane; i < W_s; i += 32) {
        const int ii = dir ? W_s - 1 - i : i;
        v = max(v, y + hi16(cp[ii]));
      }
      v = warp_max(v);
      if (lane == 0) {
        atomicMax(&S.newmax[cfg], v);
        atomicAdd(&S.work, (unsigned long long)W_s);
      }
    }
    __syncthreads();
    // ---- hierarchical selection -----------------------------------
    if (tid == 0) {
      const int32_t sw0 = max(S.fmax, S.newmax[0]), sw1 = max(S.fmax, S.newmax[1]);
      int d0 = sw1 < sw0 ? 1 : 0;                 // ties -> left to right
      if (no_bal) d0 = S.rows & 1;                // static alternation (ablation)
      int cfg = d0;
      if (knee_ok) {
        const int32_t sk0 = max(S.conc_max, S.newmax[2]), sk1 = max(S.conc_max, S.newmax[3]);
        const int d1 = sk1 < sk0 ? 1 : 0;
        const int32_t swk = max(S.fmax, S.newmax[2 + d1]);
        if (swk <= (d0 ? sw1 : sw0) - 1) cfg = 2 + d1;  // "at least marginally smaller"
      }
      S.sel_cfg = cfg;
      S.fmax = max(S.fmax, S.newmax[cfg]);
      S.knee_key = 0ull;
    }
    __syncthreads();
    // ---- commit: F <- max(F, Y + BottomEdge); record placements ------------
    const int cfg = S.sel_cfg;
    const int f = cfg >> 1, dir = cfg & 1;
    const int hc = f ? hc1 : hc0;
    const int32_t a_f = f ? ka : 0, b_f = f ? kb : Wp;
    const int32_t endS = S.end_cfg[cfg];
    for (int s = rs + wid; s <= endS; s += kNW) {
      const int32_t W_s = wd[s];
      const int32_t xl = hc ? xs1[s] : xs0[s];
      const int32_t X = dir ? b_f - xl - W_s : a_f + xl;
      const uint32_t* cp = col + colofs[s];
      const int32_t y = __ldcg(&Yc[(int64_t)cfg * n + s]);
      for (int i = lane; i < W_s; i += 32) {
        const int ii = dir ? W_s - 1 - i : i;
        atomicMax(&F[X + i], y + hi16(cp[ii]));
      }
      if (lane == 0) {
        Xo[s] = X;
        Yo[s] = y;
        mir[s] = (uint8_t)dir;
        atomicAdd(&S.work, (unsigned long long)W_s);
      }
    }
    // ---- FindKnee after an atlas-fold row -----------
    if (f == 0 && !no_bal) {
      for (int t = rs + tid; t < endS; t += kNT) {
        const int64_t d = (int64_t)hsorted[t] - hsorted[t + 1];
        if (10 * d >= (int64_t)pp.H * TABI_UNITS && 5 * d >= hsorted[t]) {
          const unsigned long long key =
              ((unsigned long long)d << 32) | (unsigned long long)(0x7fffffff - t);
          atomicMax(&S.knee_key, key);
        }
      }
    }
    __syncthreads();
    if (tid == 0) {
      S.rows++;
      if (f == 1) S.knee_rows++;
      if (f == 0 && !no_bal) {
        if (S.knee_key != 0ull) {
          const int t = 0x7fffffff - (int)(S.knee_key & 0xffffffffull);
          S.knee_valid = 1;
          S.knee_ltr = dir == 0;
          S.knee_left = Xo[t];
          S.knee_right = Xo[t] + wd[t];
          S.knees_found++;
        } else {
          S.knee_valid = 0;
        }
      }
      if (S.fmax > Hp) S.fail = 1;  // overflow below the atlas bottom
      S.row_start = endS + 1;
    }
    __syncthreads();
  }
  if (tid == 0) {
    cands[m - 1] = Cand{S.fail ? 0 : 1, S.fmax, S.rows, S.knees_found, S.knee_rows, 0, 0, -1};
    atomicAdd(&st->work_pack, S.work);
  }
}

// K5: the largest successful m ("return the largest scale and packing
// that succeed"), then every chart's placement in input order.
__global__ void select_kernel(PackParams pp, const int32_t* __restrict__ perm,
                              const uint8_t* __restrict__ pose, const int32_t* __restrict__ wd_all,
                              const int32_t* __restrict__ hd_all, const int32_t* __restrict__ Xo,
                              const int32_t* __restrict__ Yo, const uint8_t* __restrict__ mir,
                              const Cand* __restrict__ cands, tabi_placement* out, Status* st) {
  __shared__ int32_t win;
  if (st->bad_chart != INT32_MAX || st->capacity) return;
  if (threadIdx.x == 0) {
    int32_t w = 0;
    for (int m = pp.M; m >= 1; m--)
      if (cands[m - 1].success) { w = m; break; }
    win = w;
    if (blockIdx.x == 0) st->winner = w;
  }
  __syncthreads();
  const int32_t m = win;
  if (m == 0) return;
  const int s = blockIdx.x * blockDim.x + threadIdx.x;
  if (s >= pp.n) return;
  const int64_t b = (int64_t)(m - 1) * pp.n + s;
  const int c = perm[s];
  const uint8_t ps = pose[c];
  tabi_placement p;
  p.tx = Xo[b];
  p.ty = Yo[b];
  p.scale_num = m;
  p.scale_den = pp.M;
  p.box_w = wd_all[b] - 2 * pp.g;
  p.box_h = hd_all[b] - 2 * pp.g;
  p.rot90 = ps & 1;
  p.flip_x = (ps >> 1) & 1;
  p.flip_y = (ps >> 2) & 1;
  p.mirror_x = mir[b];
  p.mode = 0;
  p.pad[0] = p.pad[1] = p.pad[2] = 0;
  out[c] = p;
}

}  // namespace

void launch_pack(const PackParams& pp, const int32_t* colofs, const int32_t* rowofs,
                 const uint32_t* dcol, const uint32_t* drow, const int32_t* wd, const int32_t* hd,
                 const int32_t* off, const uint8_t* lockbits, const int32_t* hsorted,
                 const int32_t* cand_bad, int32_t* scratch, int64_t pair_cap, int32_t* X,
                 int32_t* Y, uint8_t* mir, Cand* cands, Status* st, cudaStream_t s) {
  const size_t smem = sizeof(int32_t) * (size_t)pp.Wp;
  static bool attr = false;
  if (!attr) {
    cudaFuncSetAttribute(pack_kernel, cudaFuncAttributeMaxDynamicSharedMemorySize,
                         (int)(sizeof(int32_t) * (TABI_MAX_ATLAS_SIDE + 2 * 64 + 8)));
    attr = true;
  }
  pack_kernel<<<pp.M, kNT, smem, s>>>(pp, colofs, rowofs, dcol, drow, wd, hd, off, lockbits,
                                      hsorted, cand_bad, scratch, pair_cap, X, Y, mir, cands, st);
}

void launch_select(const PackParams& pp, const Proxies& P, const int32_t* perm, const int32_t* wd,
                   const int32_t* hd, const int32_t* X, const int32_t* Y, const uint8_t* mir,
                   const Cand* cands, tabi_placement* out, Status* st, cudaStream_t s) {
  const int blocks = (pp.n + 255) / 256;
  select_kernel<<<blocks, 256, 0, s>>>(pp, perm, P.pose, wd, hd, X, Y, mir, cands, out, st);
}

}  // namespace tabi
