// band_kernel.cuh — device code of the band path (band_path.cu includes it twice:
// namespace bd0 with kDbg = kProf = false, the production kernel, bd1 with kDbg =
// true, the barrier-serialised debug mode MLMCP_BAND_SYNC=1, bd2 with the cycle
// probes of MLMCP_BAND_PROF=1 — compile-time switches, because runtime checks
// between the phases of a PCG iteration split its straight-line code and cost
// 3% of the kernel).  Not a standalone header.
struct Th {
  int x, k, rank, gy0;
  int vb;          // exchange-buffer index of row 0
  int sb;          // slot of row 0 (row r: sb + r * kTX)
  int gr0;         // global point index of row 0 (row r: gr0 + r * wd)
  int wd;
  uint32_t okm;    // valid rows (bit r)
  uint32_t cl[kR / 4];  // point classes of the rows (bytes)
  __device__ bool ok(int r) const { return (okm >> r) & 1u; }
  __device__ bool chg(int r) const { return (okm >> (16 + r)) & 1u; }   // class(r) != class(r-1)
  // no class change among the rows 1 .. kR-3 (the rows 0, 1, kR-2, kR-1 always
  // load their own stencil row: the domain's first / last rows and a region
  // boundary at a band edge land there, so nearly every strip qualifies)
  __device__ bool mid_uniform() const { return ((okm >> 18) & ((1u << (kR - 4)) - 1u)) == 0u; }
  // row r reloads its stencil row: always at the strip's ends, in between only
  // where the class changes (kCheck; compiled out for mid-uniform strips)
  template <bool kCheck>
  __device__ bool reload(int r) const {
    return r <= 1 || r >= kR - 2 || (kCheck && chg(r));
  }
  __device__ int row(int r) const { return gr0 + r * wd; }
  __device__ int slot(int r) const { return sb + r * kTX; }
  __device__ int cls(int r) const { return (cl[r >> 2] >> (8 * (r & 3))) & 255; }
};

struct Sh {
  double* VA;     // exchange: a_n (the final state for the energy)
  double* VC;     // exchange: u (PCG), two buffers by iteration parity
  double* X;      // [kSlots] x
  uint64_t* mb;   // mbarriers: [0..1] halo rows of VC[b], [2..3] CTA partials of
                  // RED[b], [4] halo rows of VA
  uint32_t ph;    // wait parity bits of the five mbarriers
  int hb;         // VC buffer of the current iteration
  double* PF;     // [kMaxSig][2R-1] strip factors, one set per strip signature
  double* XS;     // [2][kSlots] the task's periodic steady state (Re, Im), predictor only
  double* TAB;    // [rC][kTabW]
  double* RED;    // [2][4][kCS] CTA partials of every CTA, [4][kWarps] warp partials
  int par;
  bool pf_tab;    // the source profile is a function of the point class (TAB[c][15])
  __device__ double* vc() const { return VC + hb * kV; }
};

// strip block-Jacobi: L D L^T of the thread's 16-row tridiagonal block.  The
// factors depend only on the strip's signature — the classes of its rows and
// which rows exist — and a band has a handful of those (region interiors,
// region boundary columns, the domain's first / last column), so one set per
// signature is kept in shared memory ([sig][2R-1]: lf_0..lf_14, di_0..di_15)
// and the threads of a signature read it by broadcast.
struct Pc {
  const double* f;   // the thread's signature's set
  __device__ double lf(int r) const { return f[r]; }
  __device__ double di(int r) const { return f[kR - 1 + r]; }
};

// Region-linear stencils (A = M + dt K, M and K; slot order SW, S, W, C, E, N, NE)
// of one point class: stream_path.cu's region_stencil arithmetic.
__device__ __forceinline__ void bd_stencil(const BdArgs& a, const double2* sp, uint32_t key,
                                           double dt, double (&A)[7], double (&Mo)[7],
                                           double (&Ko)[7]) {
  const uint32_t code = key & 0x00ffffffu, mask = key >> 24;
  double2 p[6];
#pragma unroll
  for (int e = 0; e < 6; ++e) p[e] = sp[(code >> (4 * e)) & 15u];
  double m = 0.0, k = 0.0;
#pragma unroll
  for (int e = 0; e < 6; ++e) {
    m = __dadd_rn(m, __dmul_rn(p[e].x, a.rmw[e]));
    k = __dadd_rn(k, __dmul_rn(p[e].y, a.rkw[e]));
  }
  Mo[3] = m;
  Ko[3] = k;
  A[3] = op_entry(m, k, dt);
  const int slot[6] = {0, 1, 2, 4, 5, 6};
  const int e0[6] = {0, 0, 1, 2, 3, 4}, e1[6] = {1, 2, 3, 4, 5, 5};
  const int cw[6] = {10, 8, 6, 6, 8, 10};
#pragma unroll
  for (int c = 0; c < 6; ++c) {
    const bool ok = (mask >> c) & 1u;
    double mm = 0.0, kk = 0.0;
    if (ok) {
      mm = __dadd_rn(__dadd_rn(0.0, __dmul_rn(p[e0[c]].x, a.rmw[cw[c]])),
                     __dmul_rn(p[e1[c]].x, a.rmw[cw[c] + 1]));
      kk = __dadd_rn(__dadd_rn(0.0, __dmul_rn(p[e0[c]].y, a.rkw[cw[c]])),
                     __dmul_rn(p[e1[c]].y, a.rkw[cw[c] + 1]));
    }
    Mo[slot[c]] = mm;
    Ko[slot[c]] = kk;
    A[slot[c]] = ok ? op_entry(mm, kk, dt) : 0.0;
  }
}

// Exchange of a vector with the neighbouring bands: own rows by plain stores,
// the band's first / last row into the neighbouring CTAs' halo rows by
// st.async counted on their mbarrier `mi` (one arrival: this CTA's expected
// byte count).  bd_xwait (after a __syncthreads) waits for both halo rows.
// Every buffer is rewritten only after the CTAs reading it have contributed to
// an all-reduce in between, so no neighbour still reads what is overwritten.
__device__ __forceinline__ void bd_xissue(const Th& th, const double (&v)[kR], double* V, Sh& sh,
                                          int mi) {
  if (kDbg) bd_sync();
  uint64_t* mb = sh.mb + mi;
  MLMCP_DCHECK(th.vb - kLD - 1 >= 0 && th.vb + kR * kLD + 1 < kV);
#pragma unroll
  for (int r = 0; r < kR; ++r) V[th.vb + r * kLD] = v[r];
  if ((kNS == 1 || th.k == 0) && th.rank > 0)
    st_async(bd_mapa(bd_smem(V + (kHB + 1) * kLD + th.x + 1), th.rank - 1), v[0],
             bd_mapa(bd_smem(mb), th.rank - 1));
  if ((kNS == 1 || th.k == kNS - 1) && th.rank < kCS - 1)
    st_async(bd_mapa(bd_smem(V + th.x + 1), th.rank + 1), v[kR - 1],
             bd_mapa(bd_smem(mb), th.rank + 1));
  if (threadIdx.x == 0)
    mb_expect(mb, 8u * kTX * ((th.rank > 0 ? 1u : 0u) + (th.rank < kCS - 1 ? 1u : 0u)));
}
__device__ __forceinline__ void bd_xwait(Sh& sh, int mi) {
  mb_wait(sh.mb + mi, (sh.ph >> mi) & 1u);
  sh.ph ^= 1u << mi;
  if (kDbg) bd_sync();
}

// bd_xissue for a vector whose own rows are already in V: the band's edge rows
// are read back from V and sent to the neighbours
__device__ __forceinline__ void bd_xsend(const Th& th, double* V, Sh& sh, int mi) {
  if (kDbg) bd_sync();
  uint64_t* mb = sh.mb + mi;
  if ((kNS == 1 || th.k == 0) && th.rank > 0)
    st_async(bd_mapa(bd_smem(V + (kHB + 1) * kLD + th.x + 1), th.rank - 1), V[th.vb],
             bd_mapa(bd_smem(mb), th.rank - 1));
  if ((kNS == 1 || th.k == kNS - 1) && th.rank < kCS - 1)
    st_async(bd_mapa(bd_smem(V + th.x + 1), th.rank + 1), V[th.vb + (kR - 1) * kLD],
             bd_mapa(bd_smem(mb), th.rank + 1));
  if (threadIdx.x == 0)
    mb_expect(mb, 8u * kTX * ((th.rank > 0 ? 1u : 0u) + (th.rank < kCS - 1 ? 1u : 0u)));
}

// u into the next of the two PCG exchange buffers; the halo rows are waited for
// later (bd_xwait(sh, sh.hb)), after the rows that do not need them
__device__ __forceinline__ void bd_exchange_begin(const Th& th, const double (&v)[kR], Sh& sh) {
  sh.hb ^= 1;
  bd_xissue(th, v, sh.vc(), sh, sh.hb);
  __syncthreads();
}

// Calls f(r, nb) with the 7 neighbour values (SW, S, W, C, E, N, NE) of each of
// the thread's rows in turn; W / E columns are read from the exchange buffer
// row by row (few live registers), C / N / S from v.
template <class F>
__device__ __forceinline__ void bd_rows(const Th& th, const double (&v)[kR], const double* V,
                                        F&& f) {
  const int b = th.vb;
  double sw = V[b - kLD - 1], so = V[b - kLD];
  double w = V[b - 1], e = V[b + 1];
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const double en = V[b + (r + 1) * kLD + 1];               // E of row r+1 = NE of row r
    const double wn = r < kR - 1 ? V[b + (r + 1) * kLD - 1] : 0.0;
    const double nb[7] = {sw, so, w, v[r], e, r < kR - 1 ? v[r + 1] : V[b + kR * kLD], en};
    f(r, nb);
    sw = w;
    so = v[r];
    w = wn;
    e = en;
  }
}

// bd_rows with the thread's own column (C, N, S) read from V as well
template <class F>
__device__ __forceinline__ void bd_rows_s(const Th& th, const double* V, F&& f) {
  const int b = th.vb;
  double sw = V[b - kLD - 1], so = V[b - kLD];
  double w = V[b - 1], c = V[b], e = V[b + 1];
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const double en = V[b + (r + 1) * kLD + 1];
    const double cn = V[b + (r + 1) * kLD];
    const double wn = r < kR - 1 ? V[b + (r + 1) * kLD - 1] : 0.0;
    const double nb[7] = {sw, so, w, c, e, cn, en};
    f(r, nb);
    sw = w;
    so = c;
    w = wn;
    c = cn;
    e = en;
  }
}

// A stencil row held in registers across the rows of a strip: a thread's rows
// almost always share one point class (region interiors; the class changes at
// the domain's first / last row and on region boundaries), so the row is
// reloaded only where Th::chg marks a change (bit 16 + r of okm) instead of
// four shared-memory loads per row.  The row's seven coefficients (16-byte
// aligned in the class table) times the neighbours, summed in
// tile_iter_kernel's order.
struct Row7 {
  double2 t01, t23, t45;
  double t6;
  __device__ __forceinline__ void load(const double* T) {
    t01 = *reinterpret_cast<const double2*>(T);
    t23 = *reinterpret_cast<const double2*>(T + 2);
    t45 = *reinterpret_cast<const double2*>(T + 4);
    t6 = T[6];
  }
  __device__ __forceinline__ double dot(const double (&nb)[7]) const {
    double acc0 = t23.y * nb[3], acc1 = t01.x * nb[0];
    acc0 = fma(t01.y, nb[1], acc0);
    acc1 = fma(t23.x, nb[2], acc1);
    acc0 = fma(t45.x, nb[4], acc0);
    acc1 = fma(t45.y, nb[5], acc1);
    acc0 = fma(t6, nb[6], acc0);
    return acc0 + acc1;
  }
};

// out = A v for a v just handed to bd_exchange_begin: the rows 1 .. kR-2 of
// the strip need no other band's values and are formed while the neighbouring
// CTAs' halo rows are still in flight; rows 0 and kR-1 follow the wait.  Per
// row the same doubles in the same order as bd_apply.
template <bool kCheck>
__device__ __forceinline__ void bd_apply_mid(const Th& th, const Sh& sh, const double (&v)[kR],
                                             double (&out)[kR]) {
  const double* V = sh.vc();
  const int b = th.vb;
  Row7 row;
  {
    double sw = V[b - 1], so = v[0];
    double w = V[b + kLD - 1], e = V[b + kLD + 1];
#pragma unroll
    for (int r = 1; r < kR - 1; ++r) {
      if (th.reload<kCheck>(r)) row.load(sh.TAB + th.cls(r) * kTabW);
      const double en = V[b + (r + 1) * kLD + 1];
      const double wn = V[b + (r + 1) * kLD - 1];
      const double nb[7] = {sw, so, w, v[r], e, v[r + 1], en};
      out[r] = row.dot(nb);
      sw = w;
      so = v[r];
      w = wn;
      e = en;
    }
  }
}

__device__ __forceinline__ void bd_apply_overlap(const Th& th, Sh& sh, const double (&v)[kR],
                                                 double (&out)[kR]) {
  const double* V = sh.vc();
  const int b = th.vb;
  if (th.mid_uniform()) bd_apply_mid<false>(th, sh, v, out);
  else bd_apply_mid<true>(th, sh, v, out);
  Row7 row;
  bd_xwait(sh, sh.hb);
  {
    row.load(sh.TAB + th.cls(0) * kTabW);
    const double nb[7] = {V[b - kLD - 1], V[b - kLD], V[b - 1], v[0], V[b + 1], v[1],
                          V[b + kLD + 1]};
    out[0] = row.dot(nb);
  }
  {
    constexpr int r = kR - 1;
    row.load(sh.TAB + th.cls(r) * kTabW);
    const double nb[7] = {V[b + (r - 1) * kLD - 1], v[r - 1], V[b + r * kLD - 1], v[r],
                          V[b + r * kLD + 1], V[b + kR * kLD], V[b + kR * kLD + 1]};
    out[r] = row.dot(nb);
  }
}

// out = B v, B the operator part `off` (0: A, 8: M, 16: K) of the class table
__device__ __forceinline__ void bd_apply(const Th& th, const Sh& sh, int off,
                                         const double (&v)[kR], const double* V,
                                         double (&out)[kR]) {
  Row7 row;
  const double* T0 = sh.TAB + off;
  row.load(T0 + th.cls(0) * kTabW);
  bd_rows(th, v, V, [&](int r, const double (&nb)[7]) {
    if (r > 0 && th.chg(r)) row.load(T0 + th.cls(r) * kTabW);
    out[r] = row.dot(nb);
  });
}

// z = B^-1 r, B the strip's tridiagonal block
__device__ __forceinline__ void bd_precond(const Pc& pc, const double (&r_)[kR],
                                           double (&z)[kR]) {
  double y[kR];
  y[0] = r_[0];
#pragma unroll
  for (int r = 1; r < kR; ++r) y[r] = fma(-pc.lf(r - 1), y[r - 1], r_[r]);
  z[kR - 1] = pc.di(kR - 1) * y[kR - 1];
#pragma unroll
  for (int r = kR - 2; r >= 0; --r) z[r] = fma(-pc.lf(r), z[r + 1], pc.di(r) * y[r]);
}

// Cluster all-reduce of NV <= 4 doubles: warp butterfly, the CTA's 16 warp
// partials summed in warp order, the CTA totals stored into every CTA by
// st.async and counted on the receiving CTA's mbarrier (no cluster barrier),
// the 16 CTA totals summed in rank order.  Every thread of every CTA returns
// bitwise identical totals.
template <int NV>
__device__ __forceinline__ void bd_allsum_mb(double (&v)[NV], Sh& sh, int rank) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int off = 16; off > 0; off >>= 1) {
#pragma unroll
    for (int k = 0; k < NV; ++k) v[k] += __shfl_xor_sync(0xffffffffu, v[k], off);
  }
  if (kDbg) bd_sync();
  double* wp = sh.RED + 2 * 4 * kCS;        // [4][kWarps]
  double* cp = sh.RED + sh.par * 4 * kCS;   // [4][kCS]
  uint64_t* mb = sh.mb + 2 + sh.par;
  if (lane == 0) {
#pragma unroll
    for (int k = 0; k < NV; ++k) wp[k * kWarps + warp] = v[k];
  }
  __syncthreads();
  static_assert(kWarps <= 32 && (kWarps & (kWarps - 1)) == 0 && kCS == 16, "butterfly widths");
  if (warp == 0) {
    // every group of kWarps lanes sums the warp partials in the same order
#pragma unroll
    for (int k = 0; k < NV; ++k) {
      double s = wp[k * kWarps + (lane & (kWarps - 1))];
#pragma unroll
      for (int off = kWarps / 2; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off, kWarps);
      v[k] = s;
    }
    if (lane < kCS) {
      const uint32_t dst = bd_mapa(bd_smem(cp + rank), lane);
      const uint32_t rmb = bd_mapa(bd_smem(mb), lane);
#pragma unroll
      for (int k = 0; k < NV; ++k) st_async(dst + 8u * (uint32_t)(k * kCS), v[k], rmb);
    }
    if (lane == 0) mb_expect(mb, 8u * kCS * NV);
  }
  mb_wait(mb, (sh.ph >> (2 + sh.par)) & 1u);
  sh.ph ^= 1u << (2 + sh.par);
  if (kDbg) bd_sync();
#pragma unroll
  for (int k = 0; k < NV; ++k) {
    double s = cp[k * kCS + (lane & 15)];
#pragma unroll
    for (int off = 8; off > 0; off >>= 1) s += __shfl_xor_sync(0xffffffffu, s, off, 16);
    v[k] = s;
  }
  sh.par ^= 1;
}

// The step start's stencil passes: b = M a_n + dt sin(wt) profile (a_n in VA)
// with, when kEnergy, a_n^T K a_n accumulated into e2; then r_0 = b - A x_0
// (x_0 in the current exchange frame).  M / K / A rows held across the strip
// (Row7); the M row's pad entry is the class's source profile (kPfTab), global
// loads otherwise.
template <bool kEnergy, bool kPfTab, bool kCheck>
__device__ __forceinline__ void bd_start_passes(const Th& th, const BdArgs& a, const Sh& sh,
                                                double sf, double dt, double (&bv)[kR],
                                                double (&res)[kR], double& e2) {
  {
    Row7 mrow, krow;
    double pfc = 0.0;
    bd_rows_s(th, sh.VA, [&](int r, const double (&nb)[7]) {
      if (r == 0 || th.reload<kCheck>(r)) {
        const double* Tr = sh.TAB + th.cls(r) * kTabW;
        mrow.load(Tr + 8);
        pfc = Tr[15];
        if (kEnergy) krow.load(Tr + 16);
      }
      const double mx = mrow.dot(nb);
      if (kEnergy) e2 = fma(nb[3], krow.dot(nb), e2);
      double pf = pfc;
      if (!kPfTab) pf = th.ok(r) ? __ldg(a.profile + th.row(r)) : 0.0;
      bv[r] = th.ok(r) ? __dadd_rn(mx, __dmul_rn(dt, __dmul_rn(sf, pf))) : 0.0;
    });
  }
  const double* V0 = sh.vc();
  Row7 arow;
  bd_rows_s(th, V0, [&](int r, const double (&nb)[7]) {
    if (r == 0 || th.reload<kCheck>(r)) arow.load(sh.TAB + th.cls(r) * kTabW);
    res[r] = th.ok(r) ? bv[r] - arow.dot(nb) : 0.0;
  });
}

// One implicit-Euler step.  On entry the guess phase has written a_n into
// VA's own rows and the initial guess x0 into X and into the own rows of the
// next PCG exchange buffer (sh.hb already advanced); X holds a_{n+1} on exit.
// With `energy` the step's first reduction also carries a_n^T K a_n (e_out =
// half of it).  Returns MLMCP_ST_*.
__device__ __forceinline__ int bd_ie_step(const Th& th, const BdArgs& a, Sh& sh, const Pc& pc,
                                          double sf, double dt, bool energy, double& e_out,
                                          int& iters) {
  bd_xsend(th, sh.VA, sh, 4);
  bd_xsend(th, sh.vc(), sh, sh.hb);
  __syncthreads();
  bd_xwait(sh, 4);
  bd_xwait(sh, sh.hb);
  double res[kR], u[kR], p[kR], s[kR], w[kR];
  double red[4] = {0.0, 0.0, 0.0, 0.0};
  {
    double bv[kR];
    // the two stencil passes, specialised on (energy, profile from the class
    // table): no uniform branches between the rows
    const int variant = (energy ? 4 : 0) | (sh.pf_tab ? 2 : 0) | (th.mid_uniform() ? 0 : 1);
    switch (variant) {
      case 0: bd_start_passes<false, false, false>(th, a, sh, sf, dt, bv, res, red[3]); break;
      case 1: bd_start_passes<false, false, true>(th, a, sh, sf, dt, bv, res, red[3]); break;
      case 2: bd_start_passes<false, true, false>(th, a, sh, sf, dt, bv, res, red[3]); break;
      case 3: bd_start_passes<false, true, true>(th, a, sh, sf, dt, bv, res, red[3]); break;
      case 4: bd_start_passes<true, false, false>(th, a, sh, sf, dt, bv, res, red[3]); break;
      case 5: bd_start_passes<true, false, true>(th, a, sh, sf, dt, bv, res, red[3]); break;
      case 6: bd_start_passes<true, true, false>(th, a, sh, sf, dt, bv, res, red[3]); break;
      default: bd_start_passes<true, true, true>(th, a, sh, sf, dt, bv, res, red[3]); break;
    }
    bd_precond(pc, bv, u);
#pragma unroll
    for (int r = 0; r < kR; ++r) red[2] = fma(bv[r], u[r], red[2]);
  }
  bd_precond(pc, res, u);
  bd_exchange_begin(th, u, sh);
  bd_apply_overlap(th, sh, u, w);
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    red[0] = fma(res[r], u[r], red[0]);
    red[1] = fma(w[r], u[r], red[1]);
  }
  bd_allsum_mb<4>(red, sh, th.rank);
  long long tp = kProf ? clock64() : 0;
  e_out = 0.5 * red[3];
  const double gamma = red[0];
  double delta = red[1];
  const double bnorm2 = red[2];
  if (bnorm2 == 0.0) {
#pragma unroll
    for (int r = 0; r < kR; ++r) sh.X[th.slot(r)] = 0.0;
    return MLMCP_ST_OK;
  }
  const double tol2 = a.rtol2 * bnorm2;
  if (gamma <= tol2) return MLMCP_ST_OK;
  if (!isfinite(gamma)) return MLMCP_ST_NONFINITE;
  if (!(delta > 0.0)) return MLMCP_ST_BREAKDOWN;
  double alpha = gamma * fast_rcp(delta);
  double inv_g = fast_rcp(gamma);
  double c = inv_g * (delta * inv_g);
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    p[r] = sh.vc()[th.vb + r * kLD];   // u_0 (own rows of the exchange buffer)
    s[r] = w[r];
    const int sl = th.slot(r);
    sh.X[sl] = fma(alpha, p[r], sh.X[sl]);
    res[r] = fma(-alpha, s[r], res[r]);
  }
  int it = 1;
  for (;;) {
    BD_PROF2_T0(t2);
    double red2[2] = {0.0, 0.0};
    {
      double uk[kR];
      bd_precond(pc, res, uk);
      BD_PROF2(8, t2);
      bd_exchange_begin(th, uk, sh);
      BD_PROF2(9, t2);
      bd_apply_overlap(th, sh, uk, w);
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        red2[0] = fma(res[r], uk[r], red2[0]);
        red2[1] = fma(w[r], uk[r], red2[1]);
      }
      BD_PROF2(10, t2);
    }
    bd_allsum_mb<2>(red2, sh, th.rank);
    BD_PROF2(11, t2);
    const double gnew = red2[0];
    delta = red2[1];
    if (gnew <= tol2) break;
    const double beta = gnew * inv_g;
    const double den = fma(-(gnew * gnew), c, delta);
    // one exit test per iteration (the order of the codes is the former one)
    if (!isfinite(gnew) || it >= a.max_it || !(den > 0.0)) {
      iters += it;
      return !isfinite(gnew) ? MLMCP_ST_NONFINITE
             : it >= a.max_it ? MLMCP_ST_NOCONV
                              : MLMCP_ST_BREAKDOWN;
    }
    alpha = gnew * fast_rcp(den);
    inv_g = fast_rcp(gnew);
    c = inv_g * (den * inv_g);
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      // u_k back from the exchange buffer (own rows: written only by this
      // thread), so it need not stay in registers across the reduction
      const double uk = sh.vc()[th.vb + r * kLD];
      p[r] = fma(beta, p[r], uk);
      s[r] = fma(beta, s[r], w[r]);
      const int sl = th.slot(r);
      sh.X[sl] = fma(alpha, p[r], sh.X[sl]);
      res[r] = fma(-alpha, s[r], res[r]);
    }
    BD_PROF2(12, t2);
    ++it;
  }
  iters += it;
  BD_PROF(3, tp);
  return MLMCP_ST_OK;
}

// 1/2 x^T K x of the state in X over the cluster (every thread receives it)
__device__ __forceinline__ double bd_energy(const Th& th, Sh& sh) {
  double x[kR];
#pragma unroll
  for (int r = 0; r < kR; ++r) x[r] = sh.X[th.slot(r)];
  bd_xissue(th, x, sh.VA, sh, 4);
  __syncthreads();
  bd_xwait(sh, 4);
  double kx[kR];
  bd_apply(th, sh, 16, x, sh.VA, kx);
  double v[1] = {0.0};
#pragma unroll
  for (int r = 0; r < kR; ++r) v[0] = fma(x[r], kx[r], v[0]);
  bd_allsum_mb<1>(v, sh, th.rank);
  return 0.5 * v[0];
}

__global__ void __launch_bounds__(kNT, 1) band_propagate_kernel(BdArgs a) {
  static_assert(kR % kGB == 0, "guess batches of kGB rows");
  extern __shared__ __align__(16) double smem[];
  __shared__ int live;
  __shared__ double2 sp[16];
  __shared__ double sc[5];
  cg::cluster_group cl = cg::this_cluster();
  Th th;
  th.rank = (int)cl.block_rank();
  th.x = threadIdx.x % kTX;
  th.k = threadIdx.x / kTX;
  th.gy0 = th.rank * kHB + th.k * kR;
  th.vb = (th.k * kR + 1) * kLD + th.x + 1;
  th.sb = th.k * kR * kTX + th.x;
  th.wd = a.wd;
  th.gr0 = th.gy0 * a.wd + th.x;
  th.okm = 0u;
#pragma unroll
  for (int r = 0; r < kR; ++r)
    if (th.x < a.wd && th.gy0 + r < a.gh) th.okm |= 1u << r;
  const int ti = blockIdx.x / kCS;
  const mlmcp_task t = a.tasks[ti];
  const int64_t t_start = global_ns();
  const int C = a.rC;
  Sh sh;
  sh.VA = smem;
  sh.VC = sh.VA + kV;
  sh.X = sh.VC + 2 * kV;
  sh.PF = sh.X + kSlots;
  sh.XS = sh.PF + kPF;
  sh.TAB = sh.XS + 2 * kSlots;
  sh.RED = sh.TAB + kTabW * C;
  sh.mb = reinterpret_cast<uint64_t*>(sh.RED + kRedD);
  sh.ph = 0u;
  sh.hb = 1;
#ifdef MLMCP_CHECKED
  {
    uint32_t dyn;
    asm("mov.u32 %0, %%dynamic_smem_size;" : "=r"(dyn));
    MLMCP_DCHECK((size_t)(reinterpret_cast<char*>(sh.mb + 5) - reinterpret_cast<char*>(smem)) <= dyn);
    MLMCP_DCHECK(th.gy0 * kTX + th.x + (kR - 1) * kTX < kBandPts);
    MLMCP_DCHECK(C >= 1 && C <= kMaxC && a.R >= 1 && a.R <= 16);
  }
#endif
  sh.par = 0;
  for (int i = threadIdx.x; i < 3 * kV; i += kNT) smem[i] = 0.0;
  if (threadIdx.x == 0) {
    for (int i = 0; i < 5; ++i) mb_init(sh.mb + i, 1);
    asm volatile("fence.mbarrier_init.release.cluster;\n" ::: "memory");
  }
  if (th.rank == 0 && threadIdx.x == 0) {
    const int lv = (a.active == nullptr || t.group < 0)
                       ? 1
                       : (*((volatile const int32_t*)a.active + t.group) != 0);
    for (int c = 0; c < kCS; ++c) *cl.map_shared_rank(&live, c) = lv;
  }
  if (threadIdx.x < a.R)
    sp[threadIdx.x] = reinterpret_cast<const double2*>(a.rpar)[(int64_t)t.sample * a.R + threadIdx.x];
#pragma unroll
  for (int i = 0; i < kR / 4; ++i) th.cl[i] = 0u;
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    MLMCP_DCHECK(!th.ok(r) || (th.row(r) >= 0 && th.row(r) < a.N));
    if (th.ok(r)) th.cl[r >> 2] |= (uint32_t)__ldg(a.rcls + th.row(r)) << (8 * (r & 3));
  }
#pragma unroll
  for (int r = 1; r < kR; ++r)
    if (th.cls(r) != th.cls(r - 1)) th.okm |= 1u << (16 + r);
#ifdef MLMCP_CHECKED
  for (int r = 0; r < kR; ++r) MLMCP_DCHECK(th.cls(r) < a.rC);
#endif
  bd_sync();   // zeroed buffers, region parameters and the live flag visible
  if (!live) return;   // cluster-uniform
  for (int c = threadIdx.x; c < C; c += kNT) {
    double A7[7], M7[7], K7[7];
    bd_stencil(a, sp, __ldg(a.rckey + c), t.dt, A7, M7, K7);
    double* T = sh.TAB + c * kTabW;
#pragma unroll
    for (int d = 0; d < 7; ++d) {
      T[d] = A7[d];
      T[8 + d] = M7[d];
      T[16 + d] = K7[d];
    }
    T[7] = T[15] = T[23] = 0.0;
  }
  __syncthreads();
  {
    // The source profile (dt sin(wt) profile_i in the rhs) depends only on which
    // of the point's six triangles carry the source, i.e. on its class: every
    // thread stores its points' values into their classes' M-row pad slot and
    // the step start reads it with the M row.  A class whose points disagree
    // bitwise (non-uniform element areas) keeps the global loads (CTA-wide).
    __shared__ int pf_bad;
    if (threadIdx.x == 0) pf_bad = 0;
    double pfv[kR];
#pragma unroll
    for (int r = 0; r < kR; ++r) {
      pfv[r] = th.ok(r) ? __ldg(a.profile + th.row(r)) : 0.0;
      if (th.ok(r)) sh.TAB[th.cls(r) * kTabW + 15] = pfv[r];
    }
    __syncthreads();
    bool bad = false;
#pragma unroll
    for (int r = 0; r < kR; ++r)
      if (th.ok(r) && !(sh.TAB[th.cls(r) * kTabW + 15] == pfv[r])) bad = true;
    if (bad) pf_bad = 1;
    __syncthreads();
    sh.pf_tab = pf_bad == 0;
  }
  Pc pc;   // strip block-Jacobi factors (ClOp::load's recurrence)
  {
    // the thread's strip signature: its rows' classes and validity.  The first
    // thread with a signature leads it; leaders are numbered in thread order
    // (sh.X is free until the state is loaded below: signature words, leader
    // flags and dense numbers live there meanwhile).
    uint32_t* sw = reinterpret_cast<uint32_t*>(sh.X);        // [kNT][5]
    int* lead = reinterpret_cast<int*>(sw + 5 * kNT);        // [kNT] leader thread
    int* dense = lead + kNT;                                 // [kNT] signature number of a leader
    const uint32_t mine[5] = {th.cl[0], th.cl[1], th.cl[2], th.cl[3], th.okm & 0xffffu};
#pragma unroll
    for (int k = 0; k < 5; ++k) sw[threadIdx.x * 5 + k] = mine[k];
    __syncthreads();
    int ld = threadIdx.x;
    for (int j = 0; j < (int)threadIdx.x; ++j) {
      bool same = true;
#pragma unroll
      for (int k = 0; k < 5; ++k) same = same && sw[j * 5 + k] == mine[k];
      if (same) {
        ld = j;
        break;
      }
    }
    lead[threadIdx.x] = ld;
    __syncthreads();
    if (ld == (int)threadIdx.x) {
      int n = 0;
      for (int j = 0; j < (int)threadIdx.x; ++j) n += lead[j] == j;
      dense[threadIdx.x] = n;
    }
    __syncthreads();
    const int sig = dense[ld];
    MLMCP_DCHECK(sig >= 0 && sig < kMaxSig);
    double* F = sh.PF + (sig < kMaxSig ? sig : 0) * (2 * kR - 1);
    pc.f = F;
    if (ld == (int)threadIdx.x && sig < kMaxSig) {
      double d = th.ok(0) ? sh.TAB[th.cls(0) * kTabW + 3] : 0.0;
#pragma unroll
      for (int r = 0; r < kR; ++r) {
        if (r > 0) {
          const double nprev = th.ok(r - 1) ? sh.TAB[th.cls(r - 1) * kTabW + 5] : 0.0;
          const double lf = (d != 0.0) ? nprev / d : 0.0;
          F[r - 1] = lf;
          d = (th.ok(r) ? sh.TAB[th.cls(r) * kTabW + 3] : 0.0) - lf * nprev;
        }
        F[kR - 1 + r] = (th.ok(r) && d != 0.0) ? 1.0 / d : 0.0;
      }
    }
    __syncthreads();   // factors written; sh.X free again
  }
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const double v = th.ok(r) ? __ldcg(a.xbuf + t.x_in + th.row(r)) : 0.0;
    sh.X[th.slot(r)] = v;
    if (t.traj >= 0 && th.ok(r)) a.xbuf[t.traj + th.row(r)] = v;
  }
  const bool pred = a.xss != nullptr && t.ss_slot >= 0 &&
                    !(t.flags & MLMCP_TASK_NO_EXTRAPOLATION);
  const int max_order = (t.flags & MLMCP_TASK_NO_EXTRAPOLATION) ? 0 : a.order;
  const int64_t N = a.N;
  // the thread's ring entries: slot sl, row r at rb[sl * kBandPts + r * kTX]
  double* rb = a.ring + (int64_t)ti * kRing * kBandPts + th.gy0 * kTX + th.x;
  const double* Xs = pred ? a.xss + (int64_t)t.ss_slot * 2 * N : nullptr;
  // the task's periodic steady state stays in shared memory for all its steps
  // (it was re-read from L2 in every guess: a fifth of the guess's traffic)
#pragma unroll
  for (int r = 0; r < kR; ++r) {
    const int64_t j = th.row(r);
    sh.XS[th.slot(r)] = (th.ok(r) && pred) ? __ldg(Xs + j) : 0.0;
    sh.XS[kSlots + th.slot(r)] = (th.ok(r) && pred) ? __ldg(Xs + N + j) : 0.0;
  }
  const bool sum_e = t.qoi_mode == MLMCP_QOI_SUM_ENERGY && t.qoi_slot >= 0;
  // least-squares degree of the guess: by the task's steps per period
  const int lsdeg = a.ls_on > 1 ? a.ls_on : (a.omega * t.dt * 192.0 < 6.283185307179586 ? 5 : 6);
  int iters = 0, code = MLMCP_ST_OK, fail_step = 0;
  double acc = 0.0;
  long long tq = kProf ? clock64() : 0;
  for (int step = 0; step < t.n_steps; ++step) {
    BD_PROF(4, tq);
    const int64_t g = t.k0 + step + 1;
    // the step's trigonometry once per CTA, three warps in parallel
    if (threadIdx.x == 0) sc[4] = sin(__dmul_rn(a.omega, grid_time(t.t_base, g, t.dt)));
    if (pred && threadIdx.x == 32)
      sincos(__dmul_rn(a.omega, grid_time(t.t_base, g, t.dt)), &sc[0], &sc[1]);
    if (pred && threadIdx.x == 64)
      sincos(__dmul_rn(a.omega, grid_time(t.t_base, g - 1, t.dt)), &sc[2], &sc[3]);
    __syncthreads();
    BD_PROF(0, tq);
    const double sf = sc[4];
    // guess: x0 = extrapolated transient + steady state; y_n joins the ring.
    // The weights of this step (least-squares fit or exact extrapolation, zero
    // beyond the order) are rotated onto the ring slots, ww[s] = w[(step - s)
    // & 7], so every slot index is a compile-time one; slots not yet written
    // in this task are neither loaded nor weighted.
    const int pord = min(step, max_order);
    const int cur = step & (kRing - 1);
    double w0, ww[kRing];
    uint32_t valid = 0u;
#pragma unroll
    for (int sl = 0; sl < kRing; ++sl) {
      const int q = (step - sl) & (kRing - 1);
      const double wq = (pred && pord >= 7 && a.ls_on) ? (lsdeg == 5   ? c_bd_ls58[q]
                                                          : lsdeg == 4 ? c_bd_ls48[q]
                                                                       : c_bd_ls68[q])
                        : q <= pord                    ? c_bd_extrap[pord][q]
                                                       : 0.0;
      ww[sl] = (q >= 1 && q <= pord) ? wq : 0.0;
      if (q >= 1 && q <= pord) valid |= 1u << sl;
      if (q == 0) w0 = wq;
    }
    sh.hb ^= 1;
    double* VN = sh.vc();     // the step's first exchange buffer (x0)
#pragma unroll
    for (int h = 0; h < kR; h += kGB) {
      double pv[kGB][kRing], xr[kGB], xi[kGB];   // kGB rows' loads in flight together
#pragma unroll
      for (int rr = 0; rr < kGB; ++rr) {
        const int r = h + rr;
        const bool ok = th.ok(r) && pord > 0;
        xr[rr] = sh.XS[th.slot(r)];
        xi[rr] = sh.XS[kSlots + th.slot(r)];
#pragma unroll
        for (int sl = 0; sl < kRing; ++sl)
          pv[rr][sl] = (ok && ((valid >> sl) & 1u)) ? __ldcg(rb + sl * kBandPts + r * kTX) : 0.0;
      }
#pragma unroll
      for (int rr = 0; rr < kGB; ++rr) {
        const int r = h + rr;
        const double an = sh.X[th.slot(r)];
        // straight-line per row (no branch between the unrolled rows): without
        // the predictor XS holds zeros, rows outside the grid hold zeros and
        // only skip the ring store
        const double sst = pred ? fma(xr[rr], sc[0], xi[rr] * sc[1]) : 0.0;
        const double ssn = pred ? fma(xr[rr], sc[2], xi[rr] * sc[3]) : 0.0;
        const double yn = an - ssn;
        double gv = w0 * yn;
#pragma unroll
        for (int sl = 0; sl < kRing; ++sl) gv = fma(ww[sl], pv[rr][sl], gv);
        if (th.ok(r)) rb[cur * kBandPts + r * kTX] = yn;
        const double x0 = th.ok(r) ? gv + sst : 0.0;
        sh.VA[th.vb + r * kLD] = an;
        VN[th.vb + r * kLD] = x0;
        sh.X[th.slot(r)] = x0;
      }
    }
    // the energy of a_n (the state after the previous step) rides on this
    // step's first reduction
    const bool e_now = sum_e && step > 0 && t.k0 + step > t.qoi_from;
    double e = 0.0;
    BD_PROF(1, tq);
    code = bd_ie_step(th, a, sh, pc, sf, t.dt, e_now, e, iters);
    BD_PROF(2, tq);
    if (e_now) acc += e;
    if (code != MLMCP_ST_OK) { fail_step = step; break; }
    if (t.traj >= 0) {
#pragma unroll
      for (int r = 0; r < kR; ++r)
        if (th.ok(r)) a.xbuf[t.traj + (int64_t)(step + 1) * N + th.row(r)] = sh.X[th.slot(r)];
    }
  }
  if (code == MLMCP_ST_OK && t.n_steps > 0 && sum_e && t.k0 + t.n_steps > t.qoi_from)
    acc += bd_energy(th, sh);
  if (t.x_out >= 0) {
#pragma unroll
    for (int r = 0; r < kR; ++r)
      if (th.ok(r)) a.xbuf[t.x_out + th.row(r)] = sh.X[th.slot(r)];
  }
  if (code == MLMCP_ST_OK && t.qoi_mode == MLMCP_QOI_FINAL_ENERGY && t.qoi_slot >= 0)
    acc = bd_energy(th, sh);
  if (th.rank == 0 && threadIdx.x == 0) {
    if (t.qoi_slot >= 0 && t.qoi_mode != MLMCP_QOI_NONE) a.qoi[t.qoi_slot] = acc;
    if (a.iters != nullptr && t.slot >= 0) atomicAdd(a.iters + t.slot, iters);
    add_elapsed(a.elapsed, t.slot, t_start);
    if (code != MLMCP_ST_OK) {
      write_status(a.status, t.slot, code, fail_step, t.tag, t.tag);
      if (a.active != nullptr && t.group >= 0) const_cast<int32_t*>(a.active)[t.group] = 0;
    }
  }
  bd_sync();   // no CTA leaves while another may still address its shared memory
}

