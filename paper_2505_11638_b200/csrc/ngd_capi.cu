// C-ABI of the B200 NystromNGD inner solve (include/ngd.h).
//
// Host orchestration of the CUDA kernels (ngd_jet.cu, ngd_phb2.cu, ngd_gemm.cu, ngd_chol.cu,
// ngd_trsm.cu, ngd_svd.cu, ngd_vec.cu) and the NCCL all-reduces of the point-sharded multi-GPU
// path.  Every dense product of the sketch and the factorisation runs on the in-house DMMA GEMM;
// the only library compute call left is cuSOLVER's polar SVD for ell > 512 (C5's ell = 1000:
// 0.4% of the step).  Every entry point is stream-ordered on the context's
// stream; only scalars the host policy needs (loss values, PCG report, Cholesky status) are
// copied back.
#include <cusolverDn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdarg>
#include <cstdio>
#include <cstring>
#include <memory>
#include <string>
#include <vector>

#include "../../include/ngd.h"
#include "ngd_kernels.h"

#include <atomic>
namespace ngd {
extern std::atomic<long long> g_launches;
}
using namespace ngd;

namespace {

thread_local std::string g_err;

int fail(int code, const char* fmt, ...) {
  char buf[512];
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(buf, sizeof(buf), fmt, ap);
  va_end(ap);
  g_err = buf;
  return code;
}

#define CK(x)                                                                                    \
  do {                                                                                           \
    cudaError_t e_ = (x);                                                                        \
    if (e_ != cudaSuccess) return fail(NGD_E_CUDA, "%s:%d %s: %s", __FILE__, __LINE__, #x, cudaGetErrorString(e_)); \
  } while (0)
#define CKS(x)                                                                                   \
  do {                                                                                           \
    lib_probe_before(K_SOLVER, c->stream);                                                       \
    cusolverStatus_t s_ = (x);                                                                   \
    lib_probe_after(K_SOLVER, c->stream);                                                        \
    if (s_ != CUSOLVER_STATUS_SUCCESS) return fail(NGD_E_CUDA, "%s:%d %s: cusolver status %d", __FILE__, __LINE__, #x, (int)s_); \
  } while (0)
#define CKN(x)                                                                                   \
  do {                                                                                           \
    ncclResult_t r_ = (x);                                                                       \
    if (r_ != ncclSuccess) return fail(NGD_E_NCCL, "%s:%d %s: %s", __FILE__, __LINE__, #x, ncclGetErrorString(r_)); \
  } while (0)
#define TRY(x)                 \
  do {                         \
    int rc_ = (x);             \
    if (rc_ != NGD_OK) return rc_; \
  } while (0)

inline int64_t rup(int64_t a, int64_t b) { return (a + b - 1) / b * b; }

// NGD_DEBUG_SYNC=1: synchronise and check after the marked steps (locates an asynchronous fault)
bool debug_sync() {
  static const int on = [] {
    const char* e = getenv("NGD_DEBUG_SYNC");
    return e && *e == '1' ? 1 : 0;
  }();
  return on != 0;
}
#define DSYNC(tag)                                                                                  \
  do {                                                                                              \
    if (debug_sync()) {                                                                             \
      cudaError_t e_ = cudaStreamSynchronize(c->stream);                                            \
      if (e_ != cudaSuccess) return fail(NGD_E_CUDA, "after %s: %s", tag, cudaGetErrorString(e_));  \
    }                                                                                               \
  } while (0)

// grow-only device buffer
struct Buf {
  void* p = nullptr;
  size_t bytes = 0;
  bool view = false;  // points into another Buf (never freed here)
  void set_view(void* ptr, size_t n) {
    release();
    p = ptr;
    bytes = n;
    view = true;
  }
  cudaError_t ensure(size_t n) {
    if (n <= bytes) return cudaSuccess;
    if (view) return cudaErrorInvalidValue;
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
    cudaError_t e = cudaMalloc(&p, n);
    if (e == cudaSuccess) bytes = n;
    return e;
  }
  void release() {
    if (p && !view) cudaFree(p);
    p = nullptr;
    bytes = 0;
    view = false;
  }
  double* d() const { return static_cast<double*>(p); }
};

struct PcgGraph {
  cudaGraphExec_t exec = nullptr;
  int64_t key = -1;
  long long kernels = 0;  // kernel nodes (launch accounting on replay)
};

}  // namespace

struct ngd_ctx {
  int device = 0;
  cudaStream_t stream = nullptr;
  cusolverDnHandle_t sol = nullptr;  // polar SVD for ell > 512 only
  ncclComm_t comm = nullptr;
  int rank = 0, nranks = 1;

  std::vector<int> w;  // widths
  int NL = 0, d = 0, C = 0;
  int64_t p = 0;
  std::vector<int64_t> woff, boff;
  std::vector<int> Mp_f, Kp_f, Mp_r, Kp_r, mtiles;
  std::vector<int> rowbase;  // phase-A partial rows per layer
  int rows_A = 0;

  // packed operands
  std::vector<Buf> apf, apr, vp;
  // point data
  bool have_points = false;
  Geom gm{};
  int G = 1;  // phase-B splits (max over layers)
  int Gl[kMaxLayers] = {0}, kpsl[kMaxLayers] = {0};
  RedPlan rplan{};
  Buf w_pad, off_pad, w_c, F, cot_grad, cot, metric_tmp;
  Buf wr_pad, R_pad, alpha_bar;  // residual weights, residual rows, frozen 3 kappa ubar^2
  Head head{};
  unsigned lap_mask = 0;
  std::vector<Buf> zin, dbuf;  // per layer
  Buf dseed, pre_last, zs0, zs1;
  Buf jets;  // arena behind zin / dbuf / dseed
  int force_comm = 0;  // "force_comm": build a communicator (and take the multi-rank paths) even for 1 rank
  int phb_thin[kMaxLayers] = {};  // phase B route per layer: 0 ngd_phb2.cu 64 x 64 tiles, 1 thin (N <= 16 or
                                  // M <= 16, ngd_phb2.cu), 2 wide (both >= 128) on the GEMM core (ngd_phbg.cu)
  Phb2Cache phb2_cache;           // phase B: tensor maps of this context's jets
  PhbgArgs phbg{};                // wide-layer phase B plan (n_heavy = 0: none)
  PhbgCache phbg_cache;
  PhagArgs phag{};                // wide-layer phase A plan (ngd_phag.cu; n_heavy = 0: none)
  PhagCache phag_cache;
  Buf colpart;                    // phase A column partials of the wide layers [slots][s_pad]
  int pha_gemm = 2;               // option "pha_gemm": wide layers' phase A on the GEMM core (2 auto)
  int out_pre = 2;                // option "out_pre": output layer from precontracted rows (2 auto)
  int oz_max_blocks = 1024;       // option "oz_max_blocks": point blocks per row kind in the INT8 sketch's
                                  // column-maxima pass (0 = every block)
  bool pha_on = false, out_on = false;  // routes in effect (plan_routes)
  Buf gout;                       // output layer rows G[k][pt] = sum_c dseed Zin_L (out_contract)
  std::vector<char> wide_a;       // per layer: phase A eligible for the GEMM core (both sides >= 256)
  int l2u = 1;      // option "l2u": keep the preconditioner basis U L2-persisting during PCG
  Buf u_persist;     // PCG's copy of U at a fixed address (the captured graph carries its L2 window)
  size_t jets_arena = 0;
  int use_l2_window = 1;
  int l2_window_max = 0;
  bool l2_attr_set = false;
  cudaStreamAttrValue l2_attr{};
  Buf partA, partB;
  Buf redp;         // reduction partials
  Buf counters;     // unsigned counters
  Buf scal;         // device scalars
  Buf pcgs;         // PcgState
  Buf pr, pz, pd, pad, ptmp;  // PCG vectors
  Buf ppart, pcprime;         // precond scratch
  Buf jt, smat;               // sketch scratch: Jacobian-row chunk (ld = ldp), S = J_c V
  // INT8 tensor-core (Ozaki II) sketch: residues of the A side (J_c, then J_c^T), of Omega, of S;
  // product residues; row / column exponents
  Buf oz_a, oz_b, oz_s, oz_res, oz_ea, oz_eb, oz_ep, oz_ec, oz_mx;
  int sketch_engine = 2;      // option "sketch_gemm": 0 DMMA, 1 INT8 Ozaki, 2 auto (Ozaki for large sketches)
  Buf vpad, omp, yp;          // p x ell blocks at the padded leading dimension ldp (TMA: even ld)
  Buf gwork, gscrA, gscrB;    // GEMM split-K partials; staging of operands TMA cannot address
  Buf chol_t, chol_info;      // blocked Cholesky (n > 512): off-diagonal panel, per-level status
  Buf chol_pad;               // Cholesky of an odd-ld matrix: even-ld copy
  int64_t ldp = 0;            // rup(p, 16)
  Buf fj_tab;                 // FormJ device tables
  Buf nys_m, nys_tau, nys_r, nys_ur, nys_v, nys_s, nys_work, nys_info;
  Buf svd_mix;  // FP32-presweep Jacobi scratch: V0, V1, G, A2 (4 ell^2)
  double* h_pin = nullptr;    // pinned host scalars
  cusolverDnParams_t dn_params = nullptr;
  std::vector<char> h_work;
  int svd_method = 3;
  Buf trsm_work;
  Buf chol_work;
  int last_sweeps = 0;
  int last_sweeps_f32 = 0;
  int use_graphs = 1;
  int graph_gen = 0;
  cudaStream_t cap_stream = nullptr;
  Buf pargs, px, pb;
  PcgGraph pcg_graphs[2];
  int* h_flags = nullptr;
  cudaEvent_t poll_ev[4] = {nullptr, nullptr, nullptr, nullptr};
  bool lin_valid = false;
  bool lin_frozen = false;  // linearised with a separate theta_bar

  double* S(int i) { return scal.d() + i; }
  unsigned* counter(int i) { return static_cast<unsigned*>(counters.p) + i; }
};

enum Scalar { SC_LOSS = 0, SC_FRO2 = 1, SC_SHIFT = 2, SC_TMP = 3, SC_MU = 4, SC_H1 = 5 /* 2 slots */, SC_N = 8 };

static int bind(ngd_ctx* c) {
  CK(cudaSetDevice(c->device));
  return NGD_OK;
}

static int allreduce(ngd_ctx* c, double* buf, size_t n) {
  if (!c->comm) return NGD_OK;
  CKN(ncclAllReduce(buf, buf, n, ncclDouble, ncclSum, c->comm, c->stream));
  return NGD_OK;
}

// ------------------------------- forward sweep -------------------------------
// FWD over all layers.  store=true: linearisation buffers (zin/dbuf/pre_last);
// store=false: ping-pong scratch, only the output-layer pre-activations kept.
static int forward(ngd_ctx* c, bool store) {
  const Geom& gm = c->gm;
  for (int l = 0; l < c->NL; ++l) {
    const bool last = (l == c->NL - 1);
    JetArgs a{};
    a.A = c->apf[l].d();
    a.Kp = c->Kp_f[l];
    a.K = c->w[l];
    a.M = c->w[l + 1];
    a.s_pad = gm.s_pad;
    a.bias = nullptr;  // theta bias added through the packed bias vector below
    a.n_pts_pad = gm.n_pts_pad();
    const double* src;
    double* zout;
    double* pre;
    if (store) {
      src = c->zin[l].d();
      zout = last ? nullptr : c->zin[l + 1].d();
      pre = last ? c->pre_last.d() : c->dbuf[l].d();
    } else {
      src = (l == 0) ? c->zin[0].d() : ((l & 1) ? c->zs0.d() : c->zs1.d());
      zout = last ? nullptr : ((l & 1) ? c->zs1.d() : c->zs0.d());
      pre = last ? c->pre_last.d() : nullptr;
    }
    a.B = src;
    a.z_out = zout;
    a.pre_out = pre;
    a.bias = c->apf[l].d() + (int64_t)c->Mp_f[l] * c->Kp_f[l];  // packed bias follows the packed W
    a.lap_mask = c->lap_mask;
    CK(jet_gemm_both(gm.C, FWD, a, gm.nib, gm.nbb, gm.int_cols(), c->mtiles[l], c->stream));
  }
  return NGD_OK;
}

// theta -> zero-padded operand tiles of the forward sweep (W_l with its bias row) and, for the
// reverse sweep, W_{l+1}^T: one launch
static int pack_theta(ngd_ctx* c, const double* theta, bool rev) {
  PackAll pk{};
  int e = 0;
  int64_t off = 0;
  for (int l = 0; l < c->NL; ++l) {
    pk.dst[e] = c->apf[l].d();
    pk.Mp[e] = c->Mp_f[l];
    pk.Kp[e] = c->Kp_f[l];
    pk.n_out[e] = c->w[l + 1];
    pk.n_in[e] = c->w[l];
    pk.trans[e] = 0;
    pk.woff[e] = c->woff[l];
    pk.boff[e] = c->boff[l];
    pk.start[e] = off;
    off += (int64_t)c->Mp_f[l] * c->Kp_f[l] + c->Mp_f[l];  // bias row appended after the packed matrix
    ++e;
  }
  if (rev) {
    for (int l = 0; l + 1 < c->NL; ++l) {
      pk.dst[e] = c->apr[l].d();
      pk.Mp[e] = c->Mp_r[l];
      pk.Kp[e] = c->Kp_r[l];
      pk.n_out[e] = c->w[l + 2];
      pk.n_in[e] = c->w[l + 1];
      pk.trans[e] = 1;
      pk.woff[e] = c->woff[l + 1];
      pk.boff[e] = 0;
      pk.start[e] = off;
      // no bias row: the entry ends where its matrix ends (k < mat always)
      off += (int64_t)c->Mp_r[l] * c->Kp_r[l];
      ++e;
    }
  }
  pk.start[e] = off;
  pk.n_layers = e;
  pack_all(pk, theta, nullptr, c->stream);
  CK(cudaGetLastError());
  return NGD_OK;
}

static int loss_finish(ngd_ctx* c, double* h_loss, double* F, double* cot, double* dseed = nullptr,
                       const double* alpha_bar = nullptr, double* R = nullptr) {
  const Geom& gm = c->gm;
  residual_loss(c->pre_last.d(), gm, c->head, c->wr_pad.d(), c->off_pad.d(), alpha_bar, F, R, cot, dseed,
                c->redp.d(), c->counter(0), c->S(SC_LOSS), c->stream);
  TRY(allreduce(c, c->S(SC_LOSS), 1));
  if (h_loss) {
    CK(cudaMemcpyAsync(c->h_pin, c->S(SC_LOSS), sizeof(double), cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *h_loss = 0.5 * c->h_pin[0];
    if (!std::isfinite(*h_loss)) return fail(NGD_E_NONFINITE, "non-finite loss");
  }
  return NGD_OK;
}

// ------------------------------ phase A / B ---------------------------------
// forward packing plan of a parameter-layout vector into the phase-A layer matrices (vp)
static PackAll vp_plan(ngd_ctx* c) {
  PackAll pk{};
  pk.n_layers = c->NL;
  int64_t off = 0;
  for (int l = 0; l < c->NL; ++l) {
    pk.dst[l] = c->vp[l].d();
    pk.Mp[l] = c->Mp_f[l];
    pk.Kp[l] = c->Kp_f[l];
    pk.n_out[l] = c->w[l + 1];
    pk.n_in[l] = c->w[l];
    pk.woff[l] = c->woff[l];
    pk.boff[l] = c->boff[l];
    pk.start[l] = off;
    off += (int64_t)c->Mp_f[l] * c->Kp_f[l] + c->Mp_f[l];
  }
  pk.start[c->NL] = off;
  return pk;
}

// phase-B plan (ngd_phb2.cu), one CTA per SM: heavy tiles (both sides > 16) share 148 K-split
// items, thin tiles (input layer N = d, output layer M = 1) another 148; CTA i streams heavy item
// i and thin item i interleaved.  Wide layers run on the GEMM core (ngd_phbg.cu), the output layer
// on its precontracted rows when out_on (out_phase_b, ngd_vec.cu).
static int plan_phase_b(ngd_ctx* c) {
  const Geom& gm = c->gm;
  {
    const int kt = (int)(gm.s_pad / 16);
    int heavy = 0, thin = 0;
    PhbgArgs& pg = c->phbg;
    pg = PhbgArgs{};
    for (int l = 0; l < c->NL; ++l) {
      const int M = c->w[l + 1], N = c->w[l];
      c->phb_thin[l] = phbg_layer_ok(M, N) ? 2 : ((M <= 16 || N <= 16) ? 1 : 0);
      if (l == c->NL - 1 && c->out_on) {  // output layer from the precontracted rows (out_phase_b)
        c->phb_thin[l] = 3;
        continue;
      }
      if (c->phb_thin[l] == 2) {
        const int h = pg.n_heavy++;
        pg.M[h] = M;
        pg.N[h] = N;
        pg.tiles_n[h] = (N + 127) / 128;
        pg.item_start[h + 1] = pg.item_start[h] + ((M + 127) / 128) * pg.tiles_n[h];
        pg.off[h] = c->woff[l];
        c->phbg_cache.src_d[h] = (l == c->NL - 1) ? c->dseed.d() : c->dbuf[l].d();
        c->phbg_cache.src_z[h] = c->zin[l].d();
        continue;
      }
      (c->phb_thin[l] ? thin : heavy) += ((M + 63) / 64) * ((N + 63) / 64);
    }
    if (pg.n_heavy) {
      pg.kstages = kt;
      pg.G = phbg_splits(pg.item_start[pg.n_heavy], kt);
      pg.kps = (kt + pg.G - 1) / pg.G;
      pg.G = (kt + pg.kps - 1) / pg.kps;  // no empty splits
      pg.int_units = gm.nib * gm.C;
      pg.C = gm.C;
      pg.nib = gm.nib;
      pg.p = c->p;
      c->phbg_cache.s_pad = gm.s_pad;
    }
    const int gh = heavy ? std::max(1, std::min(kt, 148 / heavy)) : 1;
    // thin tiles alone in their launch (no heavy tile left off the GEMM core): the thin-only
    // pipeline runs several CTAs per SM, so the K splits fill all of them
    const int gt = thin ? std::max(1, std::min(kt, (heavy ? 148 : phb2_thin_only_ctas()) / thin)) : 1;
    int maxg = 0;
    c->rplan.n_layers = c->NL;
    for (int l = 0; l < c->NL; ++l) {
      const int Gl = c->phb_thin[l] == 3 ? kOutSplits : (c->phb_thin[l] == 2 ? pg.G : (c->phb_thin[l] ? gt : gh));
      c->Gl[l] = Gl;
      c->kpsl[l] = (kt + Gl - 1) / Gl;
      c->rplan.start[l] = c->woff[l];
      c->rplan.G[l] = Gl;
      maxg = std::max(maxg, Gl);
    }
    c->rplan.start[c->NL] = c->p;
    c->G = maxg;
  }
  CK(c->partB.ensure(sizeof(double) * (size_t)c->G * c->p));
  return NGD_OK;
}

// which phase-A / phase-B routes the options select for this geometry (option value 2 = auto)
static int plan_routes(ngd_ctx* c) {
  const Geom& gm = c->gm;
  const bool wide = c->phag.n_heavy > 0;
  // GEMM-core phase A (producer-warpgroup form): measured faster at C5 (C = 12: 19.6 vs 23.0 ms per
  // phase A) and at C4 (C = 4: 2.22 vs 2.27 ms; the single-role form had been slower there)
  c->pha_on = wide && (c->pha_gemm == 1 || (c->pha_gemm == 2 && gm.C >= 4));
  // precontracted output layer: its Jacobian rows (kout per point) replace a C-times larger jet
  // stream in both phases at the cost of one more launch per phase -- measured per C5 / C4 / C3
  // matvec 44.3 -> 42.6, 4.86 -> 4.76, 0.665 -> 0.652 ms, but C2 (kout S = 1.1 M) 46 -> 58 us
  const int kout = c->w[c->NL - 1];
  c->out_on = c->out_pre == 1 || (c->out_pre == 2 && (double)kout * (double)gm.s_pad >= (double)(1 << 23));
  if (c->out_on) CK(c->gout.ensure(sizeof(double) * (size_t)kout * gm.n_pts_pad()));
  // partial rows a route no longer writes must read as zero (reduce_pha sums every row)
  CK(cudaMemsetAsync(c->partA.p, 0, c->partA.bytes, c->stream));
  return plan_phase_b(c);
}

// bench evidence: algorithmic FLOPs (2 P_w S per phase) of the phase A / phase B invocations launched
// directly (graph captures are not counted: their replays are not timed per launch either)
static double g_phase_flops[2] = {0.0, 0.0};
static void count_phase(ngd_ctx* c, int which) {
  cudaStreamCaptureStatus cs = cudaStreamCaptureStatusNone;
  if (cudaStreamIsCapturing(c->stream, &cs) != cudaSuccess || cs != cudaStreamCaptureStatusNone) {
    cudaGetLastError();
    return;
  }
  double pw = 0.0;
  for (int l = 0; l < c->NL; ++l) pw += (double)c->w[l] * c->w[l + 1];
  g_phase_flops[which] += 2.0 * pw * ((double)c->gm.n_int * c->gm.C + c->gm.n_bnd);
}

// J v: pack v (unless prepacked: PCG's direction is packed by pcg_dir_pack), phase A, reduction
static int phase_a(ngd_ctx* c, const double* v, const double* w_or_null, double* cot_out, const int* skip,
                   bool prepacked = false) {
  const Geom& gm = c->gm;
  count_phase(c, 0);
  if (!prepacked) pack_all(vp_plan(c), v, skip, c->stream);
  PhaAll pa{};
  pa.n_layers = c->NL;
  pa.nib = gm.nib;
  pa.nbb = gm.nbb;
  pa.int_cols = gm.int_cols();
  const bool gemm_core = c->pha_on;
  if (gemm_core) {
    c->phag.colpart = c->colpart.d();
    c->phag.skip = skip;
    CK(phase_a_gemm(c->phag, c->phag_cache, c->stream));
  }
  int tiles = 0;
  for (int l = 0; l < c->NL; ++l) {
    JetArgs& a = pa.L[l];
    a.A = c->vp[l].d();
    a.Kp = c->Kp_f[l];
    a.K = c->w[l];
    a.M = c->w[l + 1];
    a.B = c->zin[l].d();
    a.s_pad = gm.s_pad;
    a.col0 = 0;
    a.pt0 = 0;
    a.bias = c->vp[l].d() + (int64_t)c->Mp_f[l] * c->Kp_f[l];
    a.Dk = (l == c->NL - 1) ? c->dseed.d() : c->dbuf[l].d();
    a.partA = c->partA.d() + (int64_t)c->rowbase[l] * gm.n_pts_pad();
    a.n_pts_pad = gm.n_pts_pad();
    a.skip = skip;
    pa.mtiles[l] = c->mtiles[l];
    pa.tile_start[l] = tiles;
    const bool elsewhere = (gemm_core && c->wide_a[l]) || (c->out_on && l == c->NL - 1);
    if (!elsewhere) tiles += c->mtiles[l] * (gm.nib + gm.nbb);
  }
  pa.tile_start[c->NL] = tiles;
  CK(pha_all(gm.C, pa, c->stream));
  if (gemm_core || c->out_on) {
    PhaCols rc{};
    if (gemm_core) {
      rc.colpart = c->colpart.d();
      rc.cslots = c->phag.slot0[c->phag.n_heavy - 1] + 2 * c->phag.tiles_m[c->phag.n_heavy - 1];
    }
    if (c->out_on) {
      const int l = c->NL - 1;
      rc.gout = c->gout.d();
      rc.kout = c->w[l];
      rc.vout = c->vp[l].d();
      rc.vbout = c->vp[l].d() + (int64_t)c->Mp_f[l] * c->Kp_f[l];
      rc.dseed = c->dseed.d();
    }
    reduce_pha_cols(c->partA.d(), c->rows_A, gm, rc, w_or_null, cot_out, skip, c->stream);
  } else {
    reduce_pha(c->partA.d(), c->rows_A, gm.n_pts_pad(), w_or_null, cot_out, skip, c->stream);
  }
  CK(cudaGetLastError());
  return NGD_OK;
}

static void fill_phb(ngd_ctx* c, const double* cot, const int* skip, PhbAll& pb) {
  const Geom& gm = c->gm;
  pb.n_layers = c->NL;
  int tiles = 0;
  for (int l = 0; l < c->NL; ++l) {
    PhbArgs& a = pb.L[l];
    a.D = (l == c->NL - 1) ? c->dseed.d() : c->dbuf[l].d();
    a.Z = c->zin[l].d();
    a.cvec = cot;
    a.M = c->w[l + 1];
    a.N = c->w[l];
    a.s_pad = gm.s_pad;
    a.int_cols = gm.int_cols();
    a.C = gm.C;
    a.nib = gm.nib;
    a.ktiles_total = (int)(gm.s_pad / 16);
    a.ktiles_per_split = c->kpsl[l];
    a.off = c->woff[l];
    a.part = c->partB.d();
    a.p = c->p;
    a.skip = skip;
    pb.tiles_n[l] = (a.N + 63) / 64;
    pb.tiles_m[l] = (a.M + 63) / 64;
    pb.G[l] = c->Gl[l];
    pb.tile_start[l] = tiles;
    tiles += pb.tiles_n[l] * pb.tiles_m[l] * c->Gl[l];
  }
  pb.tile_start[c->NL] = tiles;
  for (int l = 0; l < c->NL; ++l) pb.thin[l] = c->phb_thin[l];
}

// J^T cot partials of every layer into partB: wide layers on the GEMM core, the rest (thin input /
// output layers, narrow hidden layers) on the 64 x 64-tile pipeline
static int phase_b_partials(ngd_ctx* c, const double* cot, const int* skip) {
  count_phase(c, 1);
  if (c->phbg.n_heavy) {
    c->phbg.cvec = cot;
    c->phbg.part = c->partB.d();
    c->phbg.skip = skip;
    CK(phase_b_gemm(c->phbg, c->phbg_cache, c->stream));
  }
  if (c->out_on) {
    const int l = c->NL - 1;
    out_phase_b(c->gout.d(), c->dseed.d(), c->w[l], c->gm, cot, c->partB.d(), c->p, c->woff[l], c->Gl[l], skip,
                c->stream);
  }
  PhbAll pb{};
  fill_phb(c, cot, skip, pb);
  CK(phase_b2_all_layers(pb, c->phb2_cache, c->stream));
  return NGD_OK;
}

// out = J^T cot (+ mu v), all-reduced over ranks
static int phase_b_all(ngd_ctx* c, const double* cot, double mu, const double* mu_p, const double* v, double* out,
                       const int* skip) {
  TRY(phase_b_partials(c, cot, skip));
  const bool shifted = v && (mu_p || mu != 0.0);
  if (c->comm) {
    reduce_splits(c->partB.d(), c->rplan, c->p, 0.0, nullptr, nullptr, out, skip, c->stream);
    TRY(allreduce(c, out, c->p));
    if (shifted) add_scaled(out, mu, mu_p, v, c->p, skip, c->stream);
  } else {
    reduce_splits(c->partB.d(), c->rplan, c->p, mu, mu_p, shifted ? v : nullptr, out, skip, c->stream);
  }
  CK(cudaGetLastError());
  return NGD_OK;
}

static int gram_mv(ngd_ctx* c, const double* v, double mu, const double* mu_p, double* out, const int* skip) {
  TRY(phase_a(c, v, c->w_pad.d(), c->cot.d(), skip));
  TRY(phase_b_all(c, c->cot.d(), mu, mu_p, v, out, skip));
  return NGD_OK;
}

static int need_lin(ngd_ctx* c) {
  if (!c->have_points) return fail(NGD_E_STATE, "ngd_set_points has not been called");
  if (!c->lin_valid) return fail(NGD_E_STATE, "no linearisation: call ngd_linearize first");
  return NGD_OK;
}

// ------------------------------ dense products ------------------------------
// operand copy at an even leading dimension (TMA addresses 16-byte aligned rows only)
static int stage_operand(ngd_ctx* c, GemmOperand& o, int MN, int K, Buf& scr) {
  const int64_t inner = o.kmaj ? K : MN, outer = o.kmaj ? MN : K;
  const int64_t ld = rup(inner, 2);
  CK(scr.ensure(sizeof(double) * (size_t)(ld * outer)));
  CK(cudaMemcpy2DAsync(scr.p, sizeof(double) * ld, o.p, sizeof(double) * o.ld, sizeof(double) * inner, outer,
                       cudaMemcpyDeviceToDevice, c->stream));
  o.p = scr.d();
  o.ld = ld;
  return NGD_OK;
}

// C(M x N, ldc) = alpha A B [* row_scale] + beta C on the in-house DMMA GEMM (ngd_gemm.cu)
static int gemm(ngd_ctx* c, int M, int N, int K, double alpha, GemmOperand A, GemmOperand B, double beta, double* C,
                int64_t ldc, const double* row_scale = nullptr) {
  if (M <= 0 || N <= 0) return NGD_OK;
  if (!gemm_operand_ok(A, M, K)) TRY(stage_operand(c, A, M, K, c->gscrA));
  if (!gemm_operand_ok(B, N, K)) TRY(stage_operand(c, B, N, K, c->gscrB));
  const GemmPlan pl = gemm_plan(M, N, K);
  CK(c->gwork.ensure(std::max<size_t>(pl.work_bytes, 64)));
  CK(dgemm(M, N, K, alpha, A, B, beta, C, ldc, row_scale, c->gwork.d(), c->gwork.bytes, c->stream));
  return NGD_OK;
}
static inline GemmOperand kmaj(const double* p, int64_t ld) { return GemmOperand{p, ld, true}; }
static inline GemmOperand mnmaj(const double* p, int64_t ld) { return GemmOperand{p, ld, false}; }

// B <- B R^{-1} (B p x n col-major (ldb), R n x n upper (ldr)): DMMA solve kernel (ngd_trsm.cu) for
// n <= 512; above, blocked:  X1 = B1 R11^{-1},  B2 -= X1 R12 (GEMM),  X2 = B2 R22^{-1}
static int trsm_right(ngd_ctx* c, double* B, int64_t ldb, int64_t p, const double* R, int ldr, int n) {
  if (trsm_supported(n)) {
    CK(c->trsm_work.ensure(trsm_work(n)));
    CK(trsm_right_upper(B, ldb, p, R, ldr, n, c->trsm_work.d(), c->stream));
    return NGD_OK;
  }
  const int n1 = (int)rup((n + 1) / 2, 32), n2 = n - n1;
  TRY(trsm_right(c, B, ldb, p, R, ldr, n1));
  TRY(gemm(c, (int)p, n2, n1, -1.0, mnmaj(B, ldb), kmaj(R + (int64_t)n1 * ldr, ldr), 1.0, B + (int64_t)n1 * ldb,
           ldb));
  return trsm_right(c, B + (int64_t)n1 * ldb, ldb, p, R + (int64_t)n1 * ldr + n1, ldr, n2);
}

// Upper Cholesky A = U^T U in place (n x n column-major, lda; upper triangle read and written).
// One CTA (n <= 32), 8-CTA cluster (n <= 512, ngd_chol.cu), else blocked:
//   U11 = chol(A11);  U12 = U11^{-T} A12 (right solve on A12^T);  A22 -= U12^T U12 (GEMM);  U22 = chol(A22)
// *info (device) follows LAPACK: 0, or the first failing pivot + 1.
static int potrf_upper(ngd_ctx* c, double* A, int n, int lda, int* info, int depth = 0) {
  if (n > 32 && ((lda & 1) || (reinterpret_cast<uintptr_t>(A) & 15u))) {
    // the cluster kernel addresses columns as 16-byte aligned runs: factor an even-ld copy
    const int ldp = n + (n & 1);
    CK(c->chol_pad.ensure(sizeof(double) * (size_t)ldp * n));
    CK(cudaMemcpy2DAsync(c->chol_pad.p, sizeof(double) * ldp, A, sizeof(double) * lda, sizeof(double) * n, n,
                         cudaMemcpyDeviceToDevice, c->stream));
    TRY(potrf_upper(c, c->chol_pad.d(), n, ldp, info, depth));
    CK(cudaMemcpy2DAsync(A, sizeof(double) * lda, c->chol_pad.p, sizeof(double) * ldp, sizeof(double) * n, n,
                         cudaMemcpyDeviceToDevice, c->stream));
    return NGD_OK;
  }
  if (n <= 32) {
    CK(chol_upper(A, n, lda, info, c->stream));
    return NGD_OK;
  }
  if (chol_cluster_supported(n)) {
    CK(c->chol_work.ensure(sizeof(int) * 4));
    CK(chol_upper_cluster(A, n, lda, info, static_cast<int*>(c->chol_work.p), c->stream));
    return NGD_OK;
  }
  if (depth >= 8) return fail(NGD_E_SHAPE, "Cholesky of order %d too large", n);
  const int n1 = (int)rup((n + 1) / 2, 32), n2 = n - n1;
  CK(c->chol_info.ensure(sizeof(int) * 16));
  int* info2 = static_cast<int*>(c->chol_info.p) + depth;
  CK(cudaMemsetAsync(info2, 0, sizeof(int), c->stream));
  TRY(potrf_upper(c, A, n1, lda, info, depth + 1));
  DSYNC("blocked potrf: diagonal block 1");
  double* A12 = A + (int64_t)n1 * lda;
  CK(c->chol_t.ensure(sizeof(double) * (size_t)n1 * n2));
  double* T = c->chol_t.d();  // A12^T (n2 x n1)
  transpose(A12, lda, n1, n2, T, n2, c->stream);
  DSYNC("blocked potrf: transpose");
  TRY(trsm_right(c, T, n2, n2, A, lda, n1));  // T U11 = A12^T  ->  T = U12^T
  DSYNC("blocked potrf: trsm");
  transpose(T, n2, n2, n1, A12, lda, c->stream);
  TRY(gemm(c, n2, n2, n1, -1.0, kmaj(A12, lda), kmaj(A12, lda), 1.0, A12 + n1, lda));
  DSYNC("blocked potrf: gemm");
  TRY(potrf_upper(c, A12 + n1, n2, lda, info2, depth + 1));
  DSYNC("blocked potrf: diagonal block 2");
  info_combine(info, info2, n1, c->stream);
  return NGD_OK;
}

// W = A^T A for a tall p x ell column-major A (lda)
static int gram_tall(ngd_ctx* c, const double* A, int64_t lda, int64_t p, int ell, double* W) {
  return gemm(c, ell, ell, (int)p, 1.0, kmaj(A, lda), kmaj(A, lda), 0.0, W, ell);
}

// Shifted Cholesky-QR3 (Fukaya, Kannan, Nakatsukasa, Yamamoto, Yanagisawa 2020) in place:
// B (p x ell, ldb) <- Q, nys_r <- R (upper, ell x ell).  info[4..6]: the three Cholesky statuses.
static int scholqr3(ngd_ctx* c, double* B, int64_t ldb, int64_t p, int ell) {
  CK(c->nys_v.ensure(sizeof(double) * (size_t)ell * ell));
  int* info = static_cast<int*>(c->nys_info.p) + 4;
  const double shift_coef = 11.0 * ((double)p * ell + (double)ell * (ell + 1)) * 2.220446049250313e-16;
  for (int pass = 0; pass < 3; ++pass) {
    double* W = c->nys_m.d();
    TRY(gram_tall(c, B, ldb, p, ell, W));
    if (pass == 0) shift_diag(W, ell, shift_coef, c->stream);
    TRY(potrf_upper(c, W, ell, ell, info + pass));
    triu(W, ell, ell, c->stream);
    TRY(trsm_right(c, B, ldb, p, W, ell, ell));
    if (pass == 0) {
      CK(cudaMemcpyAsync(c->nys_r.d(), W, sizeof(double) * ell * ell, cudaMemcpyDeviceToDevice, c->stream));
    } else {
      // R <- R_pass R  (both upper triangular; the zero triangles multiply through exactly)
      TRY(gemm(c, ell, ell, ell, 1.0, mnmaj(W, ell), kmaj(c->nys_r.d(), ell), 0.0, c->nys_v.d(), ell));
      CK(cudaMemcpyAsync(c->nys_r.d(), c->nys_v.d(), sizeof(double) * ell * ell, cudaMemcpyDeviceToDevice, c->stream));
    }
  }
  return NGD_OK;
}

// SVD of the ell x ell matrix in nys_r by cuSOLVER's polar SVD (ell > 512): singular values -> nys_s
// (descending), U -> nys_ur.  info[2] <- its status (0 ok), h_err <- its residual estimate.
static int small_svd_polar(ngd_ctx* c, int ell, double* h_err) {
  if (!c->dn_params) CKS(cusolverDnCreateParams(&c->dn_params));
  size_t wd = 0, wh = 0;
  CKS(cusolverDnXgesvdp_bufferSize(c->sol, c->dn_params, CUSOLVER_EIG_MODE_VECTOR, 1, ell, ell, CUDA_R_64F,
                                   c->nys_r.d(), ell, CUDA_R_64F, c->nys_s.d(), CUDA_R_64F, c->nys_ur.d(), ell,
                                   CUDA_R_64F, c->nys_v.d(), ell, CUDA_R_64F, &wd, &wh));
  CK(c->nys_work.ensure(std::max<size_t>(wd, 8)));
  c->h_work.resize(std::max<size_t>(wh, 8));
  double err = 0.0;
  CKS(cusolverDnXgesvdp(c->sol, c->dn_params, CUSOLVER_EIG_MODE_VECTOR, 1, ell, ell, CUDA_R_64F, c->nys_r.d(), ell,
                        CUDA_R_64F, c->nys_s.d(), CUDA_R_64F, c->nys_ur.d(), ell, CUDA_R_64F, c->nys_v.d(), ell,
                        CUDA_R_64F, c->nys_work.p, wd, c->h_work.data(), wh, static_cast<int*>(c->nys_info.p) + 2,
                        &err));
  if (h_err) *h_err = err;
  return NGD_OK;
}

// SVD of nys_r by FP32 pre-sweeps + FP64 block Jacobi.  The FP32 one-sided Jacobi (rounds ~1.9x
// faster than FP64: half the shuffle and shared-memory traffic, FP32 pipes) runs until no rotation
// of a sweep exceeds a relative coupling of 1e-3; its rotations V32 are orthonormalised in FP64
// (two Newton-Schulz steps V <- V (3 I - V^T V) / 2: V32 is orthogonal to ~1e-5) and the FP64
// Jacobi finishes on X = R^T V0 from V = V0 -- 2-3 sweeps instead of 11 (C2 sketch, tools/probe
// sim).  Backward stable like the reference's LAPACK SVD: the product R^T V0 carries absolute
// errors ~eps ||R||, the level Cholesky-QR already leaves in R.
static int small_svd_mixed(ngd_ctx* c, int ell) {
  const int ld = ell + (ell & 1);  // even: V0 may be the FP64 phase's in-place V (vector columns)
  const size_t l2 = (size_t)ld * ell;
  CK(c->svd_mix.ensure(sizeof(double) * 4 * l2));
  CK(c->nys_info.ensure(sizeof(int) * 8));
  double* V0 = c->svd_mix.d();
  double* V1 = V0 + l2;
  double* G = V0 + 2 * l2;
  double* A2 = V0 + 3 * l2;
  int* info = static_cast<int*>(c->nys_info.p);
  static const double coupling = [] {  // NGD_SVD_F32_COUPLING: tuning override of the FP32 stopping coupling
    const char* e = getenv("NGD_SVD_F32_COUPLING");
    return e ? atof(e) : 1e-3;
  }();
  if (ld != ell) CK(cudaMemsetAsync(V0, 0, sizeof(double) * 2 * l2, c->stream));  // padding rows
  CK(jacobi_presweep_f32(c->nys_r.d(), ell, ell, V0, ld, coupling, info + 3, c->stream));
  for (int it = 0; it < 2; ++it) {  // two Newton-Schulz steps: V0 <- V0 (3 I - V0^T V0) / 2
    TRY(gemm(c, ell, ell, ell, 1.0, kmaj(V0, ld), kmaj(V0, ld), 0.0, G, ell));
    CK(cudaMemcpyAsync(V1, V0, sizeof(double) * l2, cudaMemcpyDeviceToDevice, c->stream));
    TRY(gemm(c, ell, ell, ell, -0.5, mnmaj(V0, ld), kmaj(G, ell), 1.5, V1, ld));
    std::swap(V0, V1);
  }
  // X = R^T V0 enters the kernel as A2^T, A2 = V0^T R
  TRY(gemm(c, ell, ell, ell, 1.0, kmaj(V0, ld), kmaj(c->nys_r.d(), ell), 0.0, A2, ell));
  CK(jacobi_svd_block_from(A2, ell, ell, V0, ld, c->nys_ur.d(), ell, c->nys_s.d(), info + 2, c->stream));
  return NGD_OK;
}

// L2 persisting window over the jets arena (B200: 79 MB persisting capacity, 128 MB max window)
static int set_l2_window(ngd_ctx* c, void* base, size_t bytes) {
  if (!c->use_l2_window) return NGD_OK;
  static int persist_max = -1, window_max = 0;  // device properties (one device type per process)
  if (persist_max < 0) {
    cudaDeviceProp prop;
    CK(cudaGetDeviceProperties(&prop, c->device));
    persist_max = prop.persistingL2CacheMaxSize;
    window_max = prop.accessPolicyMaxWindowSize;
    if (persist_max > 0) CK(cudaDeviceSetLimit(cudaLimitPersistingL2CacheSize, (size_t)persist_max));
  }
  c->l2_window_max = window_max;
  if (persist_max <= 0) return NGD_OK;
  cudaStreamAttrValue attr{};
  const size_t win = std::min(bytes, (size_t)std::max(c->l2_window_max, 1));
  attr.accessPolicyWindow.base_ptr = base;
  attr.accessPolicyWindow.num_bytes = win;
  attr.accessPolicyWindow.hitRatio = (float)std::min(1.0, (double)persist_max / (double)win);
  attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
  attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
  if (c->stream && cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &attr) != cudaSuccess)
    cudaGetLastError();
  if (c->cap_stream) CK(cudaStreamSetAttribute(c->cap_stream, cudaStreamAttributeAccessPolicyWindow, &attr));
  c->l2_attr = attr;
  c->l2_attr_set = true;
  return NGD_OK;
}

extern "C" {

const char* ngd_last_error(void) { return g_err.c_str(); }
int ngd_version(void) { return 1; }

int ngd_ctx_create(const int32_t* widths, int32_t n_widths, int32_t device, ngd_ctx** out) {
  if (!widths || n_widths < 2 || !out) return fail(NGD_E_SHAPE, "need at least input and output widths");
  for (int i = 0; i < n_widths; ++i)
    if (widths[i] < 1) return fail(NGD_E_SHAPE, "layer widths must be >= 1");
  if (widths[n_widths - 1] != 1) return fail(NGD_E_SHAPE, "scalar-output networks only (metric stack is scalar)");
  if (widths[0] > 10) return fail(NGD_E_SHAPE, "input dimension %d > 10 not compiled", widths[0]);
  auto* c = new ngd_ctx();
  c->device = device;
  if (cudaSetDevice(device) != cudaSuccess) {
    delete c;
    return fail(NGD_E_CUDA, "cudaSetDevice(%d) failed", device);
  }
  c->w.assign(widths, widths + n_widths);
  c->NL = n_widths - 1;
  c->d = widths[0];
  c->C = c->d + 2;
  // default head: the Laplacian metric of the Poisson problems
  c->head.coef[c->C - 1] = 1.0;
  c->lap_mask = (1u << c->d) - 1u;
  int64_t off = 0;
  c->rows_A = 0;
  for (int l = 0; l < c->NL; ++l) {
    const int nin = c->w[l], nout = c->w[l + 1];
    c->woff.push_back(off);
    off += (int64_t)nin * nout;
    c->boff.push_back(off);
    off += nout;
    c->Mp_f.push_back((int)rup(nout, 64));
    c->Kp_f.push_back((int)rup(nin, 16));
    c->mtiles.push_back((int)rup(nout, 64) / 64);
    c->wide_a.push_back(phbg_layer_ok(nout, nin) ? 1 : 0);
    if (l + 1 < c->NL) {
      c->Mp_r.push_back((int)rup(nout, 64));
      c->Kp_r.push_back((int)rup(c->w[l + 2], 16));
    } else {
      c->Mp_r.push_back(0);
      c->Kp_r.push_back(0);
    }
  }
  for (int l = 0; l < c->NL; ++l) {
    c->rowbase.push_back(c->rows_A);
    c->rows_A += c->mtiles[l];
  }
  c->p = off;
  c->ldp = rup(off, 16);
  c->apf.resize(c->NL);
  c->apr.resize(c->NL);
  c->vp.resize(c->NL);
  c->zin.resize(c->NL);
  c->dbuf.resize(c->NL);
  int rc = NGD_OK;
  auto ck = [&](cudaError_t e) {
    if (e != cudaSuccess && rc == NGD_OK) rc = fail(NGD_E_CUDA, "allocation failed: %s", cudaGetErrorString(e));
  };
  for (int l = 0; l < c->NL; ++l) {
    const size_t nf = sizeof(double) * ((size_t)c->Mp_f[l] * c->Kp_f[l] + c->Mp_f[l]);
    ck(c->apf[l].ensure(nf));
    ck(c->vp[l].ensure(nf));
    if (l + 1 < c->NL) ck(c->apr[l].ensure(sizeof(double) * (size_t)c->Mp_r[l] * c->Kp_r[l]));
  }
  ck(c->redp.ensure(sizeof(double) * 65536));  // block partials of the last-block reductions (grid <= 65536)
  ck(c->counters.ensure(sizeof(unsigned) * 64));
  ck(c->scal.ensure(sizeof(double) * SC_N));
  ck(c->pcgs.ensure(sizeof(PcgState)));
  ck(c->pargs.ensure(2 * sizeof(PrecondArgs)));
  if (rc == NGD_OK) {
    cudaMemset(c->counters.p, 0, c->counters.bytes);
    cudaMemset(c->scal.p, 0, c->scal.bytes);
    if (cudaMallocHost(&c->h_pin, 64 * sizeof(double)) != cudaSuccess) rc = fail(NGD_E_CUDA, "pinned alloc failed");
    if (cudaMallocHost(&c->h_flags, 8 * sizeof(int)) != cudaSuccess) rc = fail(NGD_E_CUDA, "pinned alloc failed");
    if (cudaStreamCreateWithFlags(&c->cap_stream, cudaStreamNonBlocking) != cudaSuccess)
      rc = fail(NGD_E_CUDA, "stream create failed");
    for (auto& e : c->poll_ev)
      if (cudaEventCreateWithFlags(&e, cudaEventDisableTiming) != cudaSuccess) rc = fail(NGD_E_CUDA, "event failed");
  }
  if (rc == NGD_OK && cusolverDnCreate(&c->sol) != CUSOLVER_STATUS_SUCCESS)
    rc = fail(NGD_E_CUDA, "cusolverDnCreate failed");
  if (rc != NGD_OK) {
    ngd_ctx_destroy(c);
    return rc;
  }
  *out = c;
  return NGD_OK;
}

int ngd_ctx_destroy(ngd_ctx* c) {
  if (!c) return NGD_OK;
  cudaSetDevice(c->device);
  if (c->stream) cudaStreamSynchronize(c->stream);
  cudaDeviceSynchronize();
  for (auto* v : {&c->apf, &c->apr, &c->vp, &c->zin, &c->dbuf})
    for (auto& b : *v) b.release();
  for (Buf* b : {&c->w_pad, &c->off_pad, &c->w_c, &c->F, &c->cot_grad, &c->cot, &c->metric_tmp, &c->dseed,
                 &c->pre_last, &c->zs0, &c->zs1, &c->partA, &c->partB, &c->redp, &c->counters, &c->scal, &c->pcgs,
                 &c->pr, &c->pz, &c->pd, &c->pad, &c->ptmp, &c->ppart, &c->pcprime, &c->jt, &c->smat, &c->fj_tab,
                 &c->nys_m, &c->nys_tau, &c->nys_r, &c->nys_ur, &c->nys_v, &c->nys_s, &c->nys_work, &c->nys_info, &c->svd_mix,
                 &c->vpad, &c->omp, &c->yp, &c->gwork, &c->gscrA, &c->gscrB, &c->chol_t, &c->chol_info, &c->chol_pad})
    b->release();
  if (c->h_pin) cudaFreeHost(c->h_pin);
  if (c->h_flags) cudaFreeHost(c->h_flags);
  for (auto& g : c->pcg_graphs)
    if (g.exec) cudaGraphExecDestroy(g.exec);
  for (auto& e : c->poll_ev)
    if (e) cudaEventDestroy(e);
  if (c->cap_stream) cudaStreamDestroy(c->cap_stream);
  for (Buf* b : {&c->pargs, &c->px, &c->pb, &c->oz_a, &c->oz_b, &c->oz_s, &c->oz_res, &c->oz_ea, &c->oz_eb, &c->oz_ep, &c->oz_ec, &c->oz_mx, &c->chol_work, &c->trsm_work, &c->jets, &c->wr_pad, &c->R_pad, &c->alpha_bar, &c->u_persist})
    b->release();
  if (c->dn_params) cusolverDnDestroyParams(c->dn_params);
  if (c->sol) cusolverDnDestroy(c->sol);
  if (c->comm) ncclCommDestroy(c->comm);
  delete c;
  return NGD_OK;
}

int ngd_ctx_set_stream(ngd_ctx* c, void* stream) {
  TRY(bind(c));
  c->stream = static_cast<cudaStream_t>(stream);
  CKS(cusolverDnSetStream(c->sol, c->stream));
  if (c->l2_attr_set && c->stream &&
      cudaStreamSetAttribute(c->stream, cudaStreamAttributeAccessPolicyWindow, &c->l2_attr) != cudaSuccess)
    cudaGetLastError();  // best effort on a caller-owned stream
  return NGD_OK;
}

int64_t ngd_param_count(const ngd_ctx* c) { return c ? c->p : -1; }

int ngd_nccl_unique_id(uint8_t* h_id) {
  ncclUniqueId id;
  CKN(ncclGetUniqueId(&id));
  static_assert(sizeof(id) == 128, "nccl id size");
  memcpy(h_id, &id, sizeof(id));
  return NGD_OK;
}

int ngd_ctx_set_comm(ngd_ctx* c, const uint8_t* h_id, int32_t rank, int32_t nranks) {
  TRY(bind(c));
  if (nranks < 1 || rank < 0 || rank >= nranks) return fail(NGD_E_SHAPE, "bad rank %d / world %d", rank, nranks);
  if (nranks == 1 && !c->force_comm) {
    c->rank = 0;
    c->nranks = 1;
    return NGD_OK;
  }
  ncclUniqueId id;
  memcpy(&id, h_id, sizeof(id));
  CKN(ncclCommInitRank(&c->comm, nranks, id, rank));
  c->rank = rank;
  c->nranks = nranks;
  return NGD_OK;
}

double ngd_phase_flops(int32_t kind) { return kind == 3 ? g_phase_flops[0] : (kind == 4 ? g_phase_flops[1] : 0.0); }

int ngd_set_points(ngd_ctx* c, int64_t n_int, const double* x_int, const double* w_int, const double* off_int,
                   int64_t n_bnd, const double* x_bnd, const double* w_bnd, const double* off_bnd) {
  return ngd_set_rows(c, n_int, x_int, w_int, w_int, off_int, n_bnd, x_bnd, w_bnd, w_bnd, off_bnd);
}

int ngd_set_rows(ngd_ctx* c, int64_t n_int, const double* x_int, const double* wm_int, const double* wr_int,
                 const double* off_int, int64_t n_bnd, const double* x_bnd, const double* wm_bnd,
                 const double* wr_bnd, const double* off_bnd) {
  TRY(bind(c));
  if (n_int < 0 || n_bnd < 0 || n_int + n_bnd == 0) return fail(NGD_E_SHAPE, "need at least one point");
  if (n_int + n_bnd > (int64_t)1 << 30) return fail(NGD_E_SHAPE, "too many points");
  Geom gm{};
  gm.d = c->d;
  gm.C = c->C;
  gm.n_int = (int)n_int;
  gm.n_bnd = (int)n_bnd;
  gm.nib = (int)((n_int + PB - 1) / PB);
  gm.nbb = (int)((n_bnd + PB - 1) / PB);
  gm.s_pad = (int64_t)gm.nib * PB * gm.C + (int64_t)gm.nbb * PB;
  c->gm = gm;
  const int npp = gm.n_pts_pad();
  const size_t col_b = sizeof(double) * gm.s_pad;
  // the linearisation's jets and adjoints (read twice per Gramian matvec) live in one arena that is
  // made an L2 persisting access-policy window on the compute streams
  int maxw = 16;
  std::vector<size_t> zoff(c->NL), doff(c->NL);
  size_t arena = 0;
  for (int l = 0; l < c->NL; ++l) {
    zoff[l] = arena;
    arena += rup(col_b * rup(c->w[l], 16), 256);
    if (l + 1 < c->NL) {
      doff[l] = arena;
      arena += rup(col_b * rup(c->w[l + 1], 16), 256);
      maxw = std::max<int>(maxw, (int)rup(c->w[l + 1], 16));
    }
  }
  const size_t soff = arena;
  arena += col_b * 16;
  for (auto& b : c->zin) b.release();
  for (auto& b : c->dbuf) b.release();
  c->dseed.release();
  CK(c->jets.ensure(arena));
  CK(cudaMemsetAsync(c->jets.p, 0, arena, c->stream));
  char* jb = static_cast<char*>(c->jets.p);
  for (int l = 0; l < c->NL; ++l) {
    c->zin[l].set_view(jb + zoff[l], col_b * rup(c->w[l], 16));
    if (l + 1 < c->NL) c->dbuf[l].set_view(jb + doff[l], col_b * rup(c->w[l + 1], 16));
  }
  c->dseed.set_view(jb + soff, col_b * 16);
  c->jets_arena = arena;
  TRY(set_l2_window(c, c->jets.p, arena));
  CK(c->pre_last.ensure(col_b * 16));
  CK(c->zs0.ensure(col_b * maxw));
  CK(c->zs1.ensure(col_b * maxw));
  CK(cudaMemsetAsync(c->zs0.p, 0, col_b * maxw, c->stream));
  CK(cudaMemsetAsync(c->zs1.p, 0, col_b * maxw, c->stream));
  for (Buf* b : {&c->w_pad, &c->off_pad, &c->F, &c->cot_grad, &c->cot, &c->wr_pad, &c->R_pad, &c->alpha_bar}) {
    CK(b->ensure(sizeof(double) * npp));
    CK(cudaMemsetAsync(b->p, 0, sizeof(double) * npp, c->stream));
  }
  CK(c->w_c.ensure(sizeof(double) * (n_int + n_bnd)));
  CK(c->metric_tmp.ensure(sizeof(double) * 2 * npp));  // also the H1 error terms
  // weights / offsets into padded point order
  if (n_int) {
    CK(cudaMemcpyAsync(c->w_pad.d(), wm_int, sizeof(double) * n_int, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->wr_pad.d(), wr_int, sizeof(double) * n_int, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->off_pad.d(), off_int, sizeof(double) * n_int, cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->w_c.d(), wm_int, sizeof(double) * n_int, cudaMemcpyDeviceToDevice, c->stream));
  }
  if (n_bnd) {
    CK(cudaMemcpyAsync(c->w_pad.d() + (int64_t)gm.nib * PB, wm_bnd, sizeof(double) * n_bnd, cudaMemcpyDeviceToDevice,
                       c->stream));
    CK(cudaMemcpyAsync(c->wr_pad.d() + (int64_t)gm.nib * PB, wr_bnd, sizeof(double) * n_bnd,
                       cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->off_pad.d() + (int64_t)gm.nib * PB, off_bnd, sizeof(double) * n_bnd,
                       cudaMemcpyDeviceToDevice, c->stream));
    CK(cudaMemcpyAsync(c->w_c.d() + n_int, wm_bnd, sizeof(double) * n_bnd, cudaMemcpyDeviceToDevice, c->stream));
  }
  init_point_data(c->zin[0].d(), c->dseed.d(), gm, x_int, x_bnd, c->stream);
  CK(cudaGetLastError());
  // phase-A partial rows and phase-B split plan
  CK(c->partA.ensure(sizeof(double) * (size_t)c->rows_A * npp));
  // phase-A plan of the wide layers (ngd_phag.cu): items (layer, n tile, m tile), two column-partial
  // rows per 128-row m tile
  {
    PhagArgs& pa = c->phag;
    pa = PhagArgs{};
    pa.tiles_n = (int)((gm.s_pad + 127) / 128);
    pa.s_pad = gm.s_pad;
    pa.int_units = gm.nib * gm.C;
    pa.C = gm.C;
    int slots = 0;
    for (int l = 0; l < c->NL; ++l) {
      if (!c->wide_a[l]) continue;
      const int h = pa.n_heavy++;
      pa.M[h] = c->w[l + 1];
      pa.Kp[h] = c->Kp_f[l];
      pa.tiles_m[h] = (pa.M[h] + 127) / 128;
      pa.item_start[h + 1] = pa.item_start[h] + pa.tiles_m[h] * pa.tiles_n;
      pa.slot0[h] = slots;
      slots += 2 * pa.tiles_m[h];
      pa.vbias[h] = c->vp[l].d() + (int64_t)c->Mp_f[l] * c->Kp_f[l];
      c->phag_cache.src_v[h] = c->vp[l].d();
      c->phag_cache.src_z[h] = c->zin[l].d();
      c->phag_cache.src_d[h] = c->dbuf[l].d();
      pa.dptr[h] = c->dbuf[l].d();
      c->phag_cache.mp[h] = c->Mp_f[l];
    }
    c->phag_cache.s_pad = gm.s_pad;
    if (slots) CK(c->colpart.ensure(sizeof(double) * (size_t)slots * gm.s_pad));
  }
  c->have_points = true;
  TRY(plan_routes(c));
  c->lin_valid = false;
  c->graph_gen++;
  return NGD_OK;
}

int ngd_set_head(ngd_ctx* c, const double* coef, int32_t n_coef, double kappa, uint32_t lap_mask) {
  if (!c) return fail(NGD_E_STATE, "null context");
  if (n_coef != c->C || c->C > kMaxC) return fail(NGD_E_SHAPE, "head needs %d coefficients, got %d", c->C, n_coef);
  if (lap_mask == 0 || (lap_mask >> c->d) != 0u) return fail(NGD_E_SHAPE, "lap_mask 0x%x is not a nonempty subset of %d coordinates", lap_mask, c->d);
  for (int i = 0; i < n_coef; ++i)
    if (!std::isfinite(coef[i])) return fail(NGD_E_SHAPE, "non-finite head coefficient");
  if (!std::isfinite(kappa)) return fail(NGD_E_SHAPE, "non-finite kappa");
  Head h{};
  for (int i = 0; i < n_coef; ++i) h.coef[i] = coef[i];
  h.kappa = kappa;
  c->head = h;
  c->lap_mask = lap_mask;
  c->lin_valid = false;
  return NGD_OK;
}

int ngd_loss(ngd_ctx* c, const double* theta, double* h_loss) {
  TRY(bind(c));
  if (!c->have_points) return fail(NGD_E_STATE, "ngd_set_points has not been called");
  TRY(pack_theta(c, theta, false));
  TRY(forward(c, false));
  return loss_finish(c, h_loss, nullptr, nullptr);
}

int ngd_h1_error(ngd_ctx* c, const double* theta, const double* exact, double* h_err) {
  TRY(bind(c));
  if (!c->have_points) return fail(NGD_E_STATE, "ngd_set_points has not been called");
  if (c->gm.n_int == 0) return fail(NGD_E_SHAPE, "H1 error needs interior points");
  const Geom& gm = c->gm;
  const int64_t n = (int64_t)gm.nib * PB;
  CK(c->metric_tmp.ensure(sizeof(double) * 2 * n));
  TRY(pack_theta(c, theta, false));
  TRY(forward(c, false));
  double* num = c->metric_tmp.d();
  double* den = num + n;
  h1_terms(c->pre_last.d(), gm, exact, num, den, c->stream);
  dot(c->w_pad.d(), num, n, c->redp.d(), c->counter(0), c->S(SC_H1), nullptr, c->stream);
  dot(c->w_pad.d(), den, n, c->redp.d(), c->counter(0), c->S(SC_H1 + 1), nullptr, c->stream);
  TRY(allreduce(c, c->S(SC_H1), 2));
  CK(cudaMemcpyAsync(c->h_pin, c->S(SC_H1), 2 * sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  if (c->h_pin[1] == 0.0) return fail(NGD_E_SHAPE, "exact solution has zero H1 norm");
  *h_err = std::sqrt(c->h_pin[0] / c->h_pin[1]);
  if (!std::isfinite(*h_err)) return fail(NGD_E_NONFINITE, "non-finite H1 error");
  return NGD_OK;
}

int ngd_loss_at(ngd_ctx* c, const double* theta, double alpha, const double* dir, double* h_loss) {
  TRY(bind(c));
  CK(c->ptmp.ensure(sizeof(double) * c->p));
  theta_minus(theta, alpha, dir, c->ptmp.d(), c->p, c->stream);
  return ngd_loss(c, c->ptmp.d(), h_loss);
}

int ngd_linearize(ngd_ctx* c, const double* theta, double* h_loss, double* d_metric) {
  return ngd_linearize_ex(c, theta, nullptr, h_loss, d_metric, nullptr);
}

int ngd_linearize_ex(ngd_ctx* c, const double* theta, const double* theta_bar, double* h_loss, double* d_metric,
                     double* d_resid) {
  TRY(bind(c));
  if (!c->have_points) return fail(NGD_E_STATE, "ngd_set_points has not been called");
  c->lin_valid = false;
  const double* alpha_bar = nullptr;
  if (theta_bar && theta_bar != theta && c->head.kappa != 0.0) {
    // metric coefficient frozen at theta_bar (gramian.py:36-40, problems.py:364-368)
    TRY(pack_theta(c, theta_bar, false));
    TRY(forward(c, false));
    frozen_alpha(c->pre_last.d(), c->gm, c->head.kappa, c->alpha_bar.d(), c->stream);
    alpha_bar = c->alpha_bar.d();
  }
  c->lin_frozen = alpha_bar != nullptr;
  TRY(pack_theta(c, theta, true));
  TRY(forward(c, true));
  TRY(loss_finish(c, h_loss, c->F.d(), c->cot_grad.d(), c->dseed.d(), alpha_bar, c->R_pad.d()));
  // reverse sweep over the jets: D_l from D_{l+1}
  const Geom& gm = c->gm;
  for (int l = c->NL - 2; l >= 0; --l) {
    JetArgs a{};
    a.A = c->apr[l].d();
    a.Kp = c->Kp_r[l];
    a.K = c->w[l + 2];
    a.M = c->w[l + 1];
    a.B = (l + 1 == c->NL - 1) ? c->dseed.d() : c->dbuf[l + 1].d();
    a.s_pad = gm.s_pad;
    a.dbuf = c->dbuf[l].d();
    a.n_pts_pad = gm.n_pts_pad();
    a.lap_mask = c->lap_mask;
    CK(jet_gemm_both(gm.C, REV, a, gm.nib, gm.nbb, gm.int_cols(), c->mtiles[l], c->stream));
  }
  // output layer precontracted once per linearisation: J_r[W_L] = sum_c dseed(r,c) Zin_L(:,(r,c))
  if (c->out_on) out_contract(c->zin[c->NL - 1].d(), c->dseed.d(), c->w[c->NL - 1], gm, c->gout.d(), c->stream);
  if (d_metric) gather_points(c->F.d(), d_metric, gm, c->stream);
  if (d_resid) gather_points(c->R_pad.d(), d_resid, gm, c->stream);
  CK(cudaGetLastError());
  c->lin_valid = true;
  return NGD_OK;
}

int ngd_loss_grad(ngd_ctx* c, double* d_grad) {
  TRY(bind(c));
  TRY(need_lin(c));
  if (c->lin_frozen) return fail(NGD_E_STATE, "gradient needs a linearisation with theta_bar == theta");
  return phase_b_all(c, c->cot_grad.d(), 0.0, nullptr, nullptr, d_grad, nullptr);
}

int ngd_jvp(ngd_ctx* c, const double* v, double* out) {
  TRY(bind(c));
  TRY(need_lin(c));
  TRY(phase_a(c, v, nullptr, c->cot.d(), nullptr));
  gather_points(c->cot.d(), out, c->gm, c->stream);
  CK(cudaGetLastError());
  return NGD_OK;
}

int ngd_vjp(ngd_ctx* c, const double* cot, double* out) {
  TRY(bind(c));
  TRY(need_lin(c));
  scatter_points(cot, c->cot.d(), c->gm, c->stream);
  return phase_b_all(c, c->cot.d(), 0.0, nullptr, nullptr, out, nullptr);
}

int ngd_gram_matvec(ngd_ctx* c, const double* v, double mu, double* out) {
  TRY(bind(c));
  TRY(need_lin(c));
  return gram_mv(c, v, mu, nullptr, out, nullptr);
}

// explicit Jacobian rows (FormJ) setup shared by the J-chunk sketch and the dense Gramian:
// chunks of whole point blocks in padded point order (padded points have w = 0); rows at the
// padded leading dimension ldp (the DMMA GEMM reads them with TMA: 16-byte aligned rows)
struct FormJPlan {
  FormJArgs fa;
  int nblk_total, bpc, max_nin, max_nout;
  int64_t R;
};

static int formj_plan(ngd_ctx* c, FormJPlan& pl) {
  const Geom& gm = c->gm;
  const int nblk_total = gm.nib + gm.nbb;
  const size_t budget = (size_t)8 << 30;  // bytes for one Jacobian chunk
  const int bpc = (int)std::max<int64_t>(1, std::min<int64_t>(nblk_total, (int64_t)(budget / (sizeof(double) * c->ldp * PB))));
  const int64_t R = (int64_t)bpc * PB;
  const size_t jbytes = sizeof(double) * (size_t)R * c->ldp;
  if (c->jt.bytes < jbytes) {
    CK(c->jt.ensure(jbytes));
    CK(cudaMemsetAsync(c->jt.p, 0, jbytes, c->stream));  // the row padding [p, ldp) stays zero
  }
  const int NL = c->NL;
  const size_t tab_bytes = NL * (2 * sizeof(double*) + 2 * sizeof(int) + sizeof(int64_t)) + 64;
  CK(c->fj_tab.ensure(tab_bytes));
  std::vector<char> h(tab_bytes, 0);
  auto** hz = reinterpret_cast<const double**>(h.data());
  auto** hd = hz + NL;
  auto* hoff = reinterpret_cast<int64_t*>(hd + NL);
  auto* hin = reinterpret_cast<int*>(hoff + NL);
  auto* hout = hin + NL;
  for (int l = 0; l < NL; ++l) {
    hz[l] = c->zin[l].d();
    hd[l] = (l == NL - 1) ? c->dseed.d() : c->dbuf[l].d();
    hoff[l] = c->woff[l];
    hin[l] = c->w[l];
    hout[l] = c->w[l + 1];
  }
  // pageable source: the copy is staged before cudaMemcpyAsync returns, so h may go out of scope
  CK(cudaMemcpyAsync(c->fj_tab.p, h.data(), tab_bytes, cudaMemcpyHostToDevice, c->stream));
  char* db = static_cast<char*>(c->fj_tab.p);
  FormJArgs fa{};
  fa.Z = reinterpret_cast<const double* const*>(db);
  fa.D = reinterpret_cast<const double* const*>(db + NL * sizeof(double*));
  fa.off = reinterpret_cast<const int64_t*>(db + 2 * NL * sizeof(double*));
  fa.n_in = reinterpret_cast<const int*>(db + 2 * NL * sizeof(double*) + NL * sizeof(int64_t));
  fa.n_out = fa.n_in + NL;
  fa.s_pad = gm.s_pad;
  fa.int_cols = gm.int_cols();
  fa.C = gm.C;
  fa.nib = gm.nib;
  fa.n_int = gm.n_int;
  fa.Jt = c->jt.d();
  fa.ldj = c->ldp;
  int max_nin = 1, max_nout = 1;
  for (int l = 0; l < NL; ++l) {
    max_nin = std::max(max_nin, c->w[l]);
    max_nout = std::max(max_nout, c->w[l + 1]);
  }
  pl.fa = fa;
  pl.nblk_total = nblk_total;
  pl.bpc = bpc;
  pl.R = R;
  pl.max_nin = max_nin;
  pl.max_nout = max_nout;
  return NGD_OK;
}

// G = J^T diag(w) J assembled densely: per chunk, Jacobian rows scaled by sqrt(w), then
// G += J_c^T J_c on the DMMA GEMM (gramian.py:138-145 assembles column by column; the spectrum
// dump of harness.py:237-266 uses it)
int ngd_gram_dense(ngd_ctx* c, double* G, int64_t ldg) {
  TRY(bind(c));
  TRY(need_lin(c));
  if (ldg < c->p) return fail(NGD_E_SHAPE, "ldg < p");
  FormJPlan pl;
  TRY(formj_plan(c, pl));
  const int p = (int)c->p;
  for (int b0 = 0; b0 < pl.nblk_total; b0 += pl.bpc) {
    const int nb = std::min(pl.bpc, pl.nblk_total - b0);
    const int64_t r = (int64_t)nb * PB;
    const int64_t q0 = (int64_t)b0 * PB;
    pl.fa.blk0 = b0;
    CK(form_j(pl.fa, nb, c->NL, pl.max_nin, pl.max_nout, c->stream));
    scale_cols_sqrt(c->jt.d(), c->ldp, r, c->w_pad.d() + q0, c->stream);
    TRY(gemm(c, p, p, (int)r, 1.0, mnmaj(c->jt.d(), c->ldp), mnmaj(c->jt.d(), c->ldp), q0 == 0 ? 0.0 : 1.0, G, ldg));
  }
  symmetrize_upper(G, c->p, ldg, c->stream);
  if (c->comm) {
    if (ldg != c->p) return fail(NGD_E_SHAPE, "multi-rank dense Gramian needs ldg == p");
    TRY(allreduce(c, G, (size_t)c->p * c->p));
  }
  CK(cudaGetLastError());
  return NGD_OK;
}

// The two sketch contractions on the INT8 tensor cores (ngd_ozaki.cu), per point chunk:
//   residues of J_c (row-scaled)  ->  S = diag(w) J_c V  (16 int8 GEMMs + CRT)
//   residues of J_c^T (column-scaled) and of S  ->  Y += J_c^T S
// V's residues are formed once per call.
static bool use_ozaki(ngd_ctx* c, int64_t ell) {
  if (c->sketch_engine == 0) return false;
  if (c->sketch_engine == 1) return true;
  return ell >= 256 && c->p >= 16384;  // measured crossover
}

static int matmat_ozaki(ngd_ctx* c, FormJPlan& pl, const GemmOperand& vop, int ell, double* Y, int64_t ldy) {
  // Two-sided scaling of J (one residue conversion per chunk serves both products):
  //   gamma_k = -floor(log2 max_all-points |J(., k)|)            (pass 0: maxima only, every chunk)
  //   rho_r   = t - 1 - floor(log2 max_k |J(r, k)| 2^gamma_k)     (per chunk, fused into formj)
  //   J'(r, k) = rint(J(r, k) 2^(rho_r + gamma_k))                [points][ldp], read K-major by
  //              S = diag(w) J_c V  and MN-major (as J_c^T) by  Y += J_c^T S
  //   V'(k, n) = rint(V(k, n) 2^(beta_n - gamma_k))   ->  S = 2^-(rho_r + beta_n) (J' V')
  //   S'(r, n) = rint(S(r, n) 2^(sigma_n - rho_r))    ->  Y = 2^-(gamma_k + sigma_n) (J'^T S')
  const int p = (int)c->p;
  const int64_t ldp = c->ldp;
  const int64_t ldr = rup(pl.R, 16);
  const int tp = std::min(oz_bits(p), oz_bits(pl.R)), tr = oz_bits(pl.R);
  const int sp = oz_splits(p);
  const int nrb = (int)((pl.R + 127) / 128), ncb = (int)((p + 127) / 128);  // J' in 128 x 128 blocks
  const int64_t pl_row = std::max(((int64_t)nrb * ncb * 16384 + 255) / 256 * 256 + 37 * 256,  // J' residue planes
                                  oz_plane(pl.R, ldp));
  const int64_t pl_v = oz_plane(ell, ldp), pl_s = oz_plane(ell, ldr);      // V', S' residue planes
  const int64_t pl_ys = oz_plane(ell, ldr), pl_yy = oz_plane(ell, ldp);    // product residues (S, Y)
  CK(c->oz_a.ensure((size_t)kOzMods * pl_row));
  CK(c->oz_b.ensure((size_t)kOzMods * pl_v));
  CK(c->oz_s.ensure((size_t)kOzMods * pl_s));
  CK(c->oz_res.ensure((size_t)kOzMods * std::max(pl_yy, sp * pl_ys)));
  CK(c->oz_ea.ensure(sizeof(int) * pl.R));
  CK(c->oz_ec.ensure(sizeof(int) * rup(p, 4)));
  CK(c->oz_eb.ensure(sizeof(int) * ell));
  CK(c->oz_ep.ensure(sizeof(int) * ell));
  CK(c->oz_mx.ensure(sizeof(long long) * (pl.R + p)));
  auto* A8 = static_cast<int8_t*>(c->oz_a.p);
  auto* B8 = static_cast<int8_t*>(c->oz_b.p);
  auto* S8 = static_cast<int8_t*>(c->oz_s.p);
  auto* R8 = static_cast<int8_t*>(c->oz_res.p);
  int* rho = static_cast<int*>(c->oz_ea.p);    // J rows (points)
  int* gam = static_cast<int*>(c->oz_ec.p);    // J columns (parameters)
  int* beta = static_cast<int*>(c->oz_eb.p);   // V columns
  int* sig = static_cast<int*>(c->oz_ep.p);    // S columns
  auto* rmax = static_cast<long long*>(c->oz_mx.p);
  auto* cmax = reinterpret_cast<unsigned long long*>(rmax + pl.R);
  // pass 0: column maxima of J (DMMA J tiles, no stores) over a strided sample of the point blocks --
  // up to kOzMaxBlocks interior and as many boundary blocks (the two row kinds differ in magnitude per
  // column).  gamma_k only balances the precision between the columns: rho_r comes from the true row
  // maxima of the prescaled chunk, so |J'| <= 2^t holds for any gamma; a column whose maximum the
  // sample misses by 2^b costs the other entries of the rows it dominates b of their t bits.
  CK(cudaMemsetAsync(cmax, 0, sizeof(unsigned long long) * p, c->stream));
  pl.fa.cmax = cmax;
  pl.fa.rmax = nullptr;
  pl.fa.no_store = 1;
  {
    const Geom& gm = c->gm;
    const int kOzMaxBlocks = c->oz_max_blocks;
    const int si = std::max(1, kOzMaxBlocks > 0 ? gm.nib / kOzMaxBlocks : 1);
    const int sb = std::max(1, kOzMaxBlocks > 0 ? gm.nbb / kOzMaxBlocks : 1);
    pl.fa.blk0 = 0;
    pl.fa.blk_stride = si;
    CK(form_j(pl.fa, (gm.nib + si - 1) / si, c->NL, pl.max_nin, pl.max_nout, c->stream));
    pl.fa.blk0 = gm.nib;
    pl.fa.blk_stride = sb;
    CK(form_j(pl.fa, (gm.nbb + sb - 1) / sb, c->NL, pl.max_nin, pl.max_nout, c->stream));
    pl.fa.blk_stride = 1;
  }
  CK(oz_exps(cmax, p, 1, gam, c->stream));  // max |J(., k)| 2^gamma_k in [1, 2)
  CK(oz_rows(vop.p, vop.ld, ell, p, tp, B8, ldp, pl_v, beta, false, c->stream, gam, -1));
  pl.fa.cmax = nullptr;
  pl.fa.rmax = rmax;
  pl.fa.cexp = gam;
  pl.fa.no_store = 0;
  for (int b0 = 0; b0 < pl.nblk_total; b0 += pl.bpc) {
    const int nb = std::min(pl.bpc, pl.nblk_total - b0);
    const int r = nb * PB;
    const int64_t q0 = (int64_t)b0 * PB;
    pl.fa.blk0 = b0;
    CK(cudaMemsetAsync(rmax, 0x80, sizeof(long long) * pl.R, c->stream));  // log-bit "empty"
    CK(form_j(pl.fa, nb, c->NL, pl.max_nin, pl.max_nout, c->stream));      // J_c + prescaled row maxima
    CK(oz_exps_log(rmax, r, tp, rho, c->stream));
    // J' in 128 x 128 blocks for the CTA-pair GEMM (contiguous TMA boxes in both products); the
    // one-CTA GEMM (option i8_pair = 0) reads the row-major form
    const int rb = g_oz_pair ? (r + 127) / 128 : 0;
    if (rb)
      CK(oz_rows_blocked(c->jt.d(), ldp, r, p, rb, ncb, rho, gam, A8, pl_row, c->stream));
    else
      CK(oz_rows(c->jt.d(), ldp, r, p, tp, A8, ldp, pl_row, rho, true, c->stream, gam, 1));
    CK(oz_i8gemm(A8, ldp, pl_row, false, r, B8, ldp, pl_v, ell, p, R8, ldr, pl_ys, c->stream, rb, ncb));
    CK(oz_crt(R8, ldr, pl_ys, r, ell, sp, rho, beta, c->w_pad.d() + q0, 1.0, 0.0, c->smat.d(), r, c->stream));
    CK(oz_rows(c->smat.d(), r, ell, r, tr, S8, ldr, pl_s, sig, false, c->stream, rho, -1));
    CK(oz_i8gemm(A8, ldp, pl_row, true, p, S8, ldr, pl_s, ell, r, R8, ldp, pl_yy, c->stream, rb, ncb));
    CK(oz_crt(R8, ldp, pl_yy, p, ell, 1, gam, sig, nullptr, 1.0, q0 == 0 ? 0.0 : 1.0, Y, ldy, c->stream));
  }
  pl.fa.rmax = nullptr;
  pl.fa.cexp = nullptr;
  return NGD_OK;
}

// Y = G V by the J-chunk formulation (gramian.py:55-61 as ell matvecs): per point
// chunk, explicit Jacobian rows J_c (formj_kernel), then on the DMMA GEMM
//   S = J_c V  (w folded into the epilogue)   and   Y += J_c^T S.
int ngd_gram_matmat(ngd_ctx* c, const double* V, int64_t ell, int64_t ldv, double* Y, int64_t ldy) {
  TRY(bind(c));
  TRY(need_lin(c));
  if (ell < 1 || ldv < c->p || ldy < c->p) return fail(NGD_E_SHAPE, "bad matmat shape");
  FormJPlan pl;
  TRY(formj_plan(c, pl));
  CK(c->smat.ensure(sizeof(double) * (size_t)pl.R * ell));
  const int p = (int)c->p;
  GemmOperand vop = kmaj(V, ldv);
  if (!gemm_operand_ok(vop, (int)ell, p)) {  // caller's odd leading dimension: one padded copy per call
    CK(c->vpad.ensure(sizeof(double) * (size_t)c->ldp * ell));
    CK(cudaMemcpy2DAsync(c->vpad.p, sizeof(double) * c->ldp, V, sizeof(double) * ldv, sizeof(double) * p, ell,
                         cudaMemcpyDeviceToDevice, c->stream));
    vop = kmaj(c->vpad.d(), c->ldp);
  }
  if (use_ozaki(c, ell)) {
    TRY(matmat_ozaki(c, pl, vop, (int)ell, Y, ldy));
  } else {
    for (int b0 = 0; b0 < pl.nblk_total; b0 += pl.bpc) {
      const int nb = std::min(pl.bpc, pl.nblk_total - b0);
      const int r = nb * PB;
      const int64_t q0 = (int64_t)b0 * PB;
      pl.fa.blk0 = b0;
      CK(form_j(pl.fa, nb, c->NL, pl.max_nin, pl.max_nout, c->stream));
      TRY(gemm(c, r, (int)ell, p, 1.0, kmaj(c->jt.d(), c->ldp), vop, 0.0, c->smat.d(), r, c->w_pad.d() + q0));
      TRY(gemm(c, p, (int)ell, r, 1.0, mnmaj(c->jt.d(), c->ldp), kmaj(c->smat.d(), r), q0 == 0 ? 0.0 : 1.0, Y, ldy));
    }
  }
  if (c->comm) {
    if (ldy != c->p) return fail(NGD_E_SHAPE, "multi-rank matmat needs ldy == p");
    TRY(allreduce(c, Y, (size_t)c->p * ell));
  }
  CK(cudaGetLastError());
  return NGD_OK;
}

int ngd_fill_gaussian(ngd_ctx* c, uint64_t seed, double* out, int64_t n) {
  TRY(bind(c));
  fill_gaussian(out, n, seed, c->stream);
  CK(cudaGetLastError());
  return NGD_OK;
}

// p x ell column-major block (ld p) <-> the context's copy at the padded leading dimension
static int to_padded(ngd_ctx* c, Buf& dst, const double* src, int64_t p, int ell) {
  const int64_t ld = rup(p, 16);
  CK(dst.ensure(sizeof(double) * (size_t)ld * ell));
  CK(cudaMemcpy2DAsync(dst.p, sizeof(double) * ld, src, sizeof(double) * p, sizeof(double) * p, ell,
                       cudaMemcpyDeviceToDevice, c->stream));
  return NGD_OK;
}
static int from_padded(ngd_ctx* c, double* dst, const Buf& src, int64_t p, int ell) {
  const int64_t ld = rup(p, 16);
  CK(cudaMemcpy2DAsync(dst, sizeof(double) * p, src.p, sizeof(double) * ld, sizeof(double) * p, ell,
                       cudaMemcpyDeviceToDevice, c->stream));
  return NGD_OK;
}

// Cholesky-QR of Omega in place: Omega <- Omega R^{-1} (once for p >= 4 ell, else twice).  Same
// orthonormal basis as the reference's Householder QR (sketch.py:75) up to column signs.
int ngd_nystrom_prepare(ngd_ctx* c, double* omega, int64_t p, int32_t ell) {
  TRY(bind(c));
  if (ell < 1 || ell > p) return fail(NGD_E_SHAPE, "rank must be in [1, %lld], got %d", (long long)p, ell);
  CK(c->nys_m.ensure(sizeof(double) * (size_t)ell * ell));
  CK(c->nys_info.ensure(sizeof(int) * 8));
  CK(cudaMemsetAsync(c->nys_info.p, 0, sizeof(int) * 8, c->stream));
  const int64_t ld = rup(p, 16);
  TRY(to_padded(c, c->omp, omega, p, ell));
  // A Gaussian p x ell block with p >= 4 ell has cond <= ~(sqrt(p)+sqrt(ell))/(sqrt(p)-sqrt(ell)) < 3, so
  // one Cholesky-QR pass is already orthonormal to O(eps cond^2); squarer blocks get a second pass.
  const int passes = (p >= 4 * (int64_t)ell) ? 1 : 2;
  for (int pass = 0; pass < passes; ++pass) {
    TRY(gram_tall(c, c->omp.d(), ld, p, ell, c->nys_m.d()));
    TRY(potrf_upper(c, c->nys_m.d(), ell, ell, static_cast<int*>(c->nys_info.p) + 1));
    TRY(trsm_right(c, c->omp.d(), ld, p, c->nys_m.d(), ell, ell));
  }
  // the potrf status is checked (no extra host sync) together with the sketch Cholesky in ngd_nystrom_finish
  return from_padded(c, omega, c->omp, p, ell);
}

// sketch.py:77-86: shift, Cholesky of Omega^T Y_nu, B = Y_nu C^{-1}, thin SVD of B
// (B = Q R by shifted Cholesky-QR3, SVD of R, U = Q U_R), eigenvalues max(s^2 - nu, 0).
// info words (device, read back with the results -- one host sync per sketch):
//   [0] sketch Cholesky  [1] Omega's Cholesky-QR  [2] SVD (Jacobi sweeps / gesvdp status)
//   [3] FP32 pre-sweeps  [4..6] the Cholesky factors of shifted Cholesky-QR3
int ngd_nystrom_finish(ngd_ctx* c, const double* omega, double* Y, int64_t p, int32_t ell, double* U_row,
                       double* eig, double* h_shift) {
  TRY(bind(c));
  if (ell < 1 || ell > p) return fail(NGD_E_SHAPE, "rank must be in [1, %lld], got %d", (long long)p, ell);
  const int64_t n = p * ell;
  const int64_t ld = rup(p, 16);
  for (Buf* b : {&c->nys_m, &c->nys_r, &c->nys_ur, &c->nys_v}) CK(b->ensure(sizeof(double) * (size_t)ell * ell));
  CK(c->nys_s.ensure(sizeof(double) * ell));
  CK(c->nys_info.ensure(sizeof(int) * 8));
  int* info = static_cast<int*>(c->nys_info.p);
  CK(cudaMemsetAsync(info + 4, 0, sizeof(int) * 3, c->stream));  // [0..3] are written by every path
  // 1. nu = eps ||Y||_F ; Y_nu = Y + nu Omega   (in the caller's Y, then one padded copy of each)
  dot(Y, Y, n, c->redp.d(), c->counter(1), c->S(SC_FRO2), nullptr, c->stream);
  add_shift(Y, omega, n, c->S(SC_FRO2), c->S(SC_SHIFT), c->stream);
  TRY(to_padded(c, c->omp, omega, p, ell));
  TRY(to_padded(c, c->yp, Y, p, ell));
  // 2. M = Omega^T Y_nu ; upper Cholesky
  TRY(gemm(c, ell, ell, (int)p, 1.0, kmaj(c->omp.d(), ld), kmaj(c->yp.d(), ld), 0.0, c->nys_m.d(), ell));
  TRY(potrf_upper(c, c->nys_m.d(), ell, ell, info));
  // 3. B = Y_nu C^{-1}
  TRY(trsm_right(c, c->yp.d(), ld, p, c->nys_m.d(), ell, ell));
  // 4. B = Q R by shifted Cholesky-QR3 (stable for cond(B) up to 1/eps)
  TRY(scholqr3(c, c->yp.d(), ld, p, ell));
  // 5. R = U_R diag(s) V^T, descending: FP32 pre-sweeps + FP64 block Jacobi in a thread-block
  //    cluster (ell <= 512), cuSOLVER's polar SVD above (or with option svd = 1)
  const bool jacobi = c->svd_method == 3 && jsvd_mixed_supported(ell) > 0;
  double svd_err = 0.0;
  if (jacobi)
    TRY(small_svd_mixed(c, ell));
  else
    TRY(small_svd_polar(c, ell, &svd_err));
  // 6. U = Q U_R  (column-major p x ell output, ld p)
  TRY(gemm(c, (int)p, ell, ell, 1.0, mnmaj(c->yp.d(), ld), kmaj(c->nys_ur.d(), ell), 0.0, U_row, p));
  eig_from_sv(c->nys_s.d(), ell, c->S(SC_SHIFT), eig, c->stream);
  CK(cudaMemcpyAsync(&c->h_pin[0], c->S(SC_SHIFT), sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaMemcpyAsync(&c->h_pin[8], info, 8 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  int hinfo[8];
  memcpy(hinfo, &c->h_pin[8], sizeof(hinfo));
  if (hinfo[1] != 0) return fail(NGD_E_CHOL, "test matrix is numerically rank deficient (potrf info %d)", hinfo[1]);
  if (hinfo[0] != 0) return fail(NGD_E_CHOL, "sketch Cholesky failed (potrf info %d)", hinfo[0]);
  for (int k = 4; k < 7; ++k)
    if (hinfo[k] != 0)
      return fail(NGD_E_CUDA, "shifted Cholesky-QR3 pass %d: Cholesky failed (info %d)", k - 4, hinfo[k]);
  if (h_shift) *h_shift = c->h_pin[0];
  c->last_sweeps = jacobi ? hinfo[2] : 0;
  c->last_sweeps_f32 = jacobi ? hinfo[3] : 0;
  // a non-converged FP64 Jacobi (or a timed-out block exchange) must not hand back a factor
  // (the FP32 pre-sweeps may stop at their sweep cap: the FP64 phase finishes the job)
  if (jacobi && (hinfo[2] <= 0 || hinfo[3] == -1000))
    return fail(NGD_E_CUDA, "small SVD: block Jacobi failed (FP64 sweeps %d, FP32 status %d)", hinfo[2], hinfo[3]);
  if (!jacobi && (hinfo[2] != 0 || !std::isfinite(svd_err)))
    return fail(NGD_E_CUDA, "small SVD: gesvdp failed (info %d, err %g)", hinfo[2], svd_err);
  CK(cudaGetLastError());
  return NGD_OK;
}

int ngd_dense_matmat(ngd_ctx* c, const double* G, int64_t p, const double* V, int64_t ell, double* Y) {
  TRY(bind(c));
  // G is a C-order (row-major) p x p matrix: Y(m, n) = sum_k G[m p + k] V[n p + k]
  return gemm(c, (int)p, (int)ell, (int)p, 1.0, kmaj(G, p), kmaj(V, p), 0.0, Y, p);
}

int ngd_precond_apply(ngd_ctx* c, const double* U, const double* eig, int32_t ell, double mu, const double* v,
                      double* out, int64_t p) {
  TRY(bind(c));
  CK(c->ppart.ensure(sizeof(double) * (size_t)precond_blocks(p) * ell));
  CK(c->pcprime.ensure(sizeof(double) * ell));
  PrecondArgs h{U, eig, mu};
  PrecondArgs* d = static_cast<PrecondArgs*>(c->pargs.p) + 1;  // slot 1: direct applies
  CK(cudaMemcpyAsync(d, &h, sizeof(h), cudaMemcpyHostToDevice, c->stream));
  CK(precond_apply(d, p, ell, v, out, c->ppart.d(), c->pcprime.d(), c->counter(10), nullptr, nullptr, 0,
                   c->redp.d(), c->stream));
  CK(cudaStreamSynchronize(c->stream));  // the host struct must outlive the copy
  return NGD_OK;
}

// One PCG iteration (krylov.py:59-81) on the device.  All scalars live in the
// PcgState; operands come from ctx-owned buffers and the PrecondArgs slot, so
// the same launch sequence can be captured once and replayed as a CUDA graph.
static int pcg_iteration(ngd_ctx* c, int64_t p, const double* dense, double mu, int ell, bool have_pre,
                         int recompute) {
  PcgState* sp = static_cast<PcgState*>(c->pcgs.p);
  const int* done = &sp->done;
  double *x = c->px.d(), *r = c->pr.d(), *z = c->pz.d(), *dv = c->pd.d(), *ad = c->pad.d(), *tmp = c->ptmp.d();
  const double* b = c->pb.d();
  double* mu_p = c->S(SC_MU);
  double* red = c->redp.d();
  // ad = (A + mu I) d ; dad = d.ad ; alpha / breakdown   (krylov.py:59-66)
  if (dense) {
    CK(gemv_rows(dense, p, dv, ad, done, c->stream));
    add_scaled(ad, mu, nullptr, dv, p, done, c->stream);
    pcg_ad(nullptr, c->rplan, p, mu_p, dv, ad, sp, 1, red, c->counter(4), c->stream);
  } else {
    TRY(phase_a(c, dv, c->w_pad.d(), c->cot.d(), done, /*prepacked=*/true));
    TRY(phase_b_partials(c, c->cot.d(), done));
    if (c->comm) {
      reduce_splits(c->partB.d(), c->rplan, p, 0.0, nullptr, nullptr, ad, done, c->stream);
      TRY(allreduce(c, ad, p));
      add_scaled(ad, 0.0, mu_p, dv, p, done, c->stream);
      pcg_ad(nullptr, c->rplan, p, mu_p, dv, ad, sp, 1, red, c->counter(4), c->stream);
    } else {
      pcg_ad(c->partB.d(), c->rplan, p, mu_p, dv, ad, sp, 0, red, c->counter(4), c->stream);
    }
  }
  // x += alpha d ; r -= alpha ad (or r = b - A x) ; ||r|| test   (krylov.py:66-74)
  pcg_update(x, r, dv, ad, p, sp, recompute, red, c->counter(5), c->stream);
  if (recompute) {
    if (dense) {
      CK(gemv_rows(dense, p, x, tmp, done, c->stream));
      add_scaled(tmp, mu, nullptr, x, p, done, c->stream);
    } else {
      TRY(gram_mv(c, x, 0.0, mu_p, tmp, done));
    }
    pcg_true_res(b, tmp, r, p, sp, 1, 0, red, c->counter(6), c->stream);
  }
  // z = P^{-1} r ; beta = r.z / rz ; d = z + beta d   (krylov.py:75-81)
  // the direction update also packs d for the next iteration's phase A (matrix-free path)
  const bool pack_next = !dense;
  if (have_pre)
    CK(precond_apply(static_cast<PrecondArgs*>(c->pargs.p), p, ell, r, z, c->ppart.d(), c->pcprime.d(),
                     c->counter(8), done, sp, 0, red, c->stream));
  else
    CK(precond_apply(nullptr, p, 0, r, z, nullptr, nullptr, c->counter(8), done, sp, 0, red, c->stream));
  if (pack_next)
    pcg_dir_pack(z, dv, vp_plan(c), sp, &c->h_flags[5], c->stream);
  else
    pcg_dir(z, dv, p, sp, &c->h_flags[5], c->stream);
  CK(cudaGetLastError());
  return NGD_OK;
}

int ngd_pcg(ngd_ctx* c, const double* dense, int64_t p, const double* b, double mu, const double* U,
            const double* eig, int32_t ell, double precond_mu, double rel_tol, int32_t maxit,
            int32_t recompute_every, double* x, ngd_solve_report* rep) {
  TRY(bind(c));
  if (!(rel_tol > 0.0 && rel_tol < 1.0)) return fail(NGD_E_SHAPE, "rel_tol must be in (0, 1), got %g", rel_tol);
  if (maxit < 1) return fail(NGD_E_SHAPE, "maxit must be >= 1");
  if (recompute_every < 1) recompute_every = 1 << 30;
  if (!dense) {
    TRY(need_lin(c));
    if (p != c->p) return fail(NGD_E_SHAPE, "expected vector of length %lld, got %lld", (long long)c->p, (long long)p);
  }
  if (p < 1) return fail(NGD_E_SHAPE, "empty system");
  for (Buf* bf : {&c->pr, &c->pz, &c->pd, &c->pad, &c->ptmp, &c->px, &c->pb}) CK(bf->ensure(sizeof(double) * p));
  const bool have_pre = (U != nullptr);
  if (have_pre) {
    CK(c->ppart.ensure(sizeof(double) * (size_t)precond_blocks(p) * ell));
    CK(c->pcprime.ensure(sizeof(double) * ell));
  }
  PcgState* sp = static_cast<PcgState*>(c->pcgs.p);
  const int* done = &sp->done;
  // every earlier solve ended with a stream synchronisation: no kernel can still write the flag
  *reinterpret_cast<volatile int*>(&c->h_flags[5]) = 0;
  // operands into stable, ctx-owned locations (graph replay needs fixed addresses).  With "l2u",
  // U is copied to a context buffer that carries an L2 persisting window for the solve: the two
  // passes over U per iteration otherwise lose it to the jets streamed by phase A and B.
  const bool l2u = have_pre && c->l2u && c->use_l2_window;
  if (l2u) {
    const size_t ub = sizeof(double) * (size_t)p * ell;
    CK(c->u_persist.ensure(ub));
    CK(cudaMemcpyAsync(c->u_persist.p, U, ub, cudaMemcpyDeviceToDevice, c->stream));
    U = c->u_persist.d();
    TRY(set_l2_window(c, c->u_persist.p, ub));
  }
  PrecondArgs hpa{U, eig, precond_mu};
  CK(cudaMemcpyAsync(c->pargs.p, &hpa, sizeof(hpa), cudaMemcpyHostToDevice, c->stream));
  c->h_pin[48] = mu;
  CK(cudaMemcpyAsync(c->S(SC_MU), &c->h_pin[48], sizeof(double), cudaMemcpyHostToDevice, c->stream));
  CK(cudaMemcpyAsync(c->pb.d(), b, sizeof(double) * p, cudaMemcpyDeviceToDevice, c->stream));
  double *xx = c->px.d(), *r = c->pr.d(), *z = c->pz.d(), *dv = c->pd.d(), *tmp = c->ptmp.d();
  // prologue: x = 0, r = b, z = P r, d = z, rz = r.z  (krylov.py:46-54)
  dot(c->pb.d(), c->pb.d(), p, c->redp.d(), c->counter(2), &sp->bb, nullptr, c->stream);
  pcg_init(sp, rel_tol, c->stream);
  pcg_start(c->pb.d(), xx, r, p, c->stream);
  CK(precond_apply(have_pre ? static_cast<PrecondArgs*>(c->pargs.p) : nullptr, p, have_pre ? ell : 0, r, z,
                   c->ppart.d(), c->pcprime.d(), c->counter(8), done, sp, 1, c->redp.d(), c->stream));
  pcg_first_dir(z, dv, p, sp, c->stream);
  if (!dense) pack_all(vp_plan(c), dv, &sp->done, c->stream);  // iterations use d prepacked

  // iterations: replay a captured CUDA graph of one iteration (Gram operator), or launch directly
  const bool use_graph = !dense && c->use_graphs;
  PcgGraph* graphs = c->pcg_graphs;
  const int64_t key = ((int64_t)c->graph_gen << 20) ^ ((int64_t)ell << 2) ^ (have_pre ? 1 : 0);
  if (use_graph) {
    for (int rec = 0; rec < 2; ++rec) {
      if (graphs[rec].exec && graphs[rec].key == key) continue;
      if (graphs[rec].exec) cudaGraphExecDestroy(graphs[rec].exec);
      graphs[rec].exec = nullptr;
      cudaStream_t saved = c->stream;
      c->stream = c->cap_stream;
      CK(cudaStreamBeginCapture(c->cap_stream, cudaStreamCaptureModeThreadLocal));
      const long long l0 = ngd::g_launches.load();
      int rc = pcg_iteration(c, p, nullptr, mu, ell, have_pre, rec);
      graphs[rec].kernels = ngd::g_launches.load() - l0;
      ngd::g_launches.fetch_sub(graphs[rec].kernels);  // counted per replay below
      cudaGraph_t g = nullptr;
      cudaError_t ce = cudaStreamEndCapture(c->cap_stream, &g);
      c->stream = saved;
      if (rc != NGD_OK) return rc;
      CK(ce);
      CK(cudaGraphInstantiate(&graphs[rec].exec, g, 0));
      cudaGraphDestroy(g);
      graphs[rec].key = key;
    }
  }
  int issued = 0;
  for (int it = 1; it <= maxit; ++it) {
    const int rec = (it % recompute_every == 0);
    if (use_graph) {
      CK(cudaGraphLaunch(graphs[rec].exec, c->stream));
      ngd::g_launches.fetch_add(graphs[rec].kernels);
    } else {
      TRY(pcg_iteration(c, p, dense, mu, ell, have_pre, rec));
    }
    ++issued;
    // stop enqueueing once the device has published 'done' (pcg_dir writes the flag to pinned host
    // memory at the end of every iteration; kernels of iterations after 'done' return at once).
    // With a communicator every iteration carries an all-reduce, so all ranks must enqueue the same
    // number of iterations: the host-timing-dependent early exit would pair one rank's final
    // true-residual all-reduce with another rank's iteration.  The device-side 'done' is identical
    // on every rank (all-reduced inputs, replicated arithmetic), so the extra iterations are no-ops.
    if (!c->comm && *reinterpret_cast<volatile int*>(&c->h_flags[5]) != 0) break;
  }
  // final true residual (krylov.py:83-88)
  CK(cudaMemcpyAsync(&c->h_flags[4], &sp->done, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  const int dn = c->h_flags[4];
  if (dn != 2) {
    if (dense) {
      CK(gemv_rows(dense, p, xx, tmp, nullptr, c->stream));
      add_scaled(tmp, mu, nullptr, xx, p, nullptr, c->stream);
    } else {
      TRY(gram_mv(c, xx, 0.0, c->S(SC_MU), tmp, nullptr));
    }
    pcg_true_res(c->pb.d(), tmp, r, p, sp, 0, 1, c->redp.d(), c->counter(6), c->stream);
  }
  CK(cudaMemcpyAsync(x, xx, sizeof(double) * p, cudaMemcpyDeviceToDevice, c->stream));
  PcgState hs;
  CK(cudaMemcpyAsync(c->h_pin + 20, sp, sizeof(PcgState), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  memcpy(&hs, c->h_pin + 20, sizeof(PcgState));
  CK(cudaGetLastError());
  if (getenv("NGD_PCG_DEBUG"))
    fprintf(stderr, "[ngd pcg] issued %d it %d iterations %d matvecs %d done %d (before final pass %d) breakdown %d rr %.3e rel %.3e dad %.3e alpha %.3e rz %.3e rz_new %.3e beta %.3e flag %d\n",
            issued, hs.it, hs.iterations, hs.matvecs, hs.done, dn, hs.breakdown, hs.rr, hs.rel, hs.dad, hs.alpha, hs.rz,
            hs.rz_new, hs.beta, c->h_flags[5]);
  if (rep) {
    if (dn == 2) {
      rep->iterations = 0;
      rep->matvecs = 0;
      rep->relative_residual = 0.0;
      rep->converged = 1;
      rep->breakdown = 0;
    } else {
      rep->iterations = hs.iterations;
      rep->matvecs = hs.matvecs;
      rep->relative_residual = hs.rel;
      rep->converged = hs.converged;
      rep->breakdown = hs.breakdown;
    }
  }
  (void)issued;
  if (l2u && c->jets_arena) TRY(set_l2_window(c, c->jets.p, c->jets_arena));  // back to the jets
  return NGD_OK;
}

int ngd_small_svd(ngd_ctx* c, const double* A, int32_t ell, double* U, double* sigma, int32_t method,
                  int32_t* h_sweeps) {
  TRY(bind(c));
  if (ell < 1) return fail(NGD_E_SHAPE, "empty matrix");
  for (Buf* b : {&c->nys_r, &c->nys_ur, &c->nys_v}) CK(b->ensure(sizeof(double) * (size_t)ell * ell));
  CK(c->nys_s.ensure(sizeof(double) * ell));
  CK(c->nys_info.ensure(sizeof(int) * 8));
  CK(cudaMemcpyAsync(c->nys_r.d(), A, sizeof(double) * ell * ell, cudaMemcpyDeviceToDevice, c->stream));
  int* info = static_cast<int*>(c->nys_info.p);
  double err = 0.0;
  if (method == 4) {
    if (jsvd_mixed_supported(ell) == 0)
      return fail(NGD_E_SHAPE, "ell = %d too large for the mixed-precision Jacobi SVD", ell);
    TRY(small_svd_mixed(c, ell));
  } else if (method == 3) {
    if (jsvd_block_supported(ell) == 0)
      return fail(NGD_E_SHAPE, "ell = %d too large for the block-exchange Jacobi SVD", ell);
    CK(jacobi_svd_block(c->nys_r.d(), ell, ell, c->nys_ur.d(), ell, c->nys_s.d(), info + 2, c->stream));
  } else if (method == 1) {
    TRY(small_svd_polar(c, ell, &err));
  } else {
    return fail(NGD_E_SHAPE, "small SVD method must be 1 (polar), 3 (block Jacobi) or 4 (FP32 + FP64 Jacobi)");
  }
  CK(cudaMemcpyAsync(U, c->nys_ur.d(), sizeof(double) * ell * ell, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemcpyAsync(sigma, c->nys_s.d(), sizeof(double) * ell, cudaMemcpyDeviceToDevice, c->stream));
  CK(cudaMemcpyAsync(&c->h_pin[56], info + 2, 2 * sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  int both[2];
  memcpy(both, &c->h_pin[56], 2 * sizeof(int));
  int sweeps = both[0];
  if (method == 1) {
    if (both[0] != 0 || !std::isfinite(err)) return fail(NGD_E_CUDA, "gesvdp failed (info %d)", both[0]);
    sweeps = 0;
  }
  if (method == 4) sweeps = both[1] * 1000 + both[0];  // FP32 pre-sweeps * 1000 + FP64 sweeps
  if (h_sweeps) *h_sweeps = sweeps;
  return NGD_OK;
}

// method 0: the factorisation the library uses (one CTA, cluster, or blocked above 512);
// 1: one-CTA kernel (n <= 160); 2: 8-CTA cluster kernel (n <= 512)
int ngd_small_cholesky(ngd_ctx* c, double* A, int32_t n, int32_t method, int32_t* h_info) {
  TRY(bind(c));
  if (n < 1) return fail(NGD_E_SHAPE, "empty matrix");
  CK(c->nys_info.ensure(sizeof(int) * 8));
  int* info = static_cast<int*>(c->nys_info.p) + 7;
  CK(cudaMemsetAsync(info, 0, sizeof(int), c->stream));
  if (method == 1) {
    if (!chol_supported(n)) return fail(NGD_E_SHAPE, "n = %d too large for the one-CTA Cholesky", n);
    CK(chol_upper(A, n, n, info, c->stream));
  } else if (method == 2) {
    if (!chol_cluster_supported(n)) return fail(NGD_E_SHAPE, "n = %d too large for the cluster Cholesky", n);
    CK(c->chol_work.ensure(sizeof(int) * 4));
    CK(chol_upper_cluster(A, n, n, info, static_cast<int*>(c->chol_work.p), c->stream));
  } else if (method == 0) {
    TRY(potrf_upper(c, A, n, n, info));
  } else {
    return fail(NGD_E_SHAPE, "Cholesky method must be 0, 1 or 2");
  }
  CK(cudaMemcpyAsync(&c->h_pin[60], info, sizeof(int), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  memcpy(h_info, &c->h_pin[60], sizeof(int));
  return NGD_OK;
}

// C = alpha op(A) op(B) + beta C on the in-house DMMA GEMM (test hook of ngd_gemm.cu): column-major
// operands; trans_a = 0: A is M x K (lda), 1: A is K x M; trans_b = 0: B is K x N, 1: B is N x K
int ngd_gemm(ngd_ctx* c, int32_t trans_a, int32_t trans_b, int32_t M, int32_t N, int32_t K, double alpha,
             const double* A, int64_t lda, const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  TRY(bind(c));
  if (M < 0 || N < 0 || K < 1) return fail(NGD_E_SHAPE, "bad GEMM shape");
  // column-major A (M x K): A(m, k) = A[k lda + m] -> MN-major; transposed: K-major
  const GemmOperand a{A, lda, trans_a != 0};
  const GemmOperand b{B, ldb, trans_b == 0};
  return gemm(c, M, N, K, alpha, a, b, beta, C, ldc);
}

// C = alpha A B + beta C on the INT8 tensor cores (Ozaki II, ngd_ozaki.cu; test hook): K-major
// operands A(m, k) = A[m lda + k], B(k, n) = B[n ldb + k] (lda, ldb multiples of 2), C column-major
int ngd_gemm_ozaki(ngd_ctx* c, int32_t M, int32_t N, int32_t K, double alpha, const double* A, int64_t lda,
                   const double* B, int64_t ldb, double beta, double* C, int64_t ldc) {
  TRY(bind(c));
  if (M < 1 || N < 1 || K < 1 || lda < K || ldb < K || ldc < M) return fail(NGD_E_SHAPE, "bad GEMM shape");
  const int64_t ldk = rup(K, 16), ldo = rup(M, 16);
  const int t = oz_bits(K), sp = oz_splits(K);
  const int64_t pa = oz_plane(M, ldk), pb = oz_plane(N, ldk), po = oz_plane(N, ldo);
  // the residue kernels stream 16-byte chunks: operands with an odd ld / unaligned base are staged once
  GemmOperand ao{A, lda, true}, bo{B, ldb, true};
  if (!gemm_operand_ok(ao, M, K)) TRY(stage_operand(c, ao, M, K, c->gscrA));
  if (!gemm_operand_ok(bo, N, K)) TRY(stage_operand(c, bo, N, K, c->gscrB));
  A = ao.p;
  lda = ao.ld;
  B = bo.p;
  ldb = bo.ld;
  CK(c->oz_a.ensure((size_t)kOzMods * pa));
  CK(c->oz_b.ensure((size_t)kOzMods * pb));
  CK(c->oz_res.ensure((size_t)kOzMods * sp * po));
  CK(c->oz_ea.ensure(sizeof(int) * M));
  CK(c->oz_eb.ensure(sizeof(int) * N));
  auto* A8 = static_cast<int8_t*>(c->oz_a.p);
  auto* B8 = static_cast<int8_t*>(c->oz_b.p);
  auto* R8 = static_cast<int8_t*>(c->oz_res.p);
  int* ea = static_cast<int*>(c->oz_ea.p);
  int* eb = static_cast<int*>(c->oz_eb.p);
  CK(oz_rows(A, lda, M, K, t, A8, ldk, pa, ea, false, c->stream));
  CK(oz_rows(B, ldb, N, K, t, B8, ldk, pb, eb, false, c->stream));
  CK(oz_i8gemm(A8, ldk, pa, false, M, B8, ldk, pb, N, K, R8, ldo, po, c->stream));
  CK(oz_crt(R8, ldo, po, M, N, sp, ea, eb, nullptr, alpha, beta, C, ldc, c->stream));
  return NGD_OK;
}

int ngd_get_stat(ngd_ctx* c, const char* key, int64_t* out) {
  if (!c || !key || !out) return fail(NGD_E_SHAPE, "bad stat query");
  if (!strcmp(key, "jacobi_sweeps")) {
    *out = c->last_sweeps;
    return NGD_OK;
  }
  if (!strcmp(key, "jacobi_sweeps_f32")) {
    *out = c->last_sweeps_f32;
    return NGD_OK;
  }
  if (!strcmp(key, "phase_b_splits")) {
    *out = c->G;
    return NGD_OK;
  }
  return fail(NGD_E_SHAPE, "unknown stat '%s'", key);
}

int ngd_set_option(ngd_ctx* c, const char* key, int64_t value) {
  if (!c || !key) return fail(NGD_E_SHAPE, "bad option");
  if (!strcmp(key, "graphs")) {
    c->use_graphs = value ? 1 : 0;
    return NGD_OK;
  }
  if (!strcmp(key, "force_comm")) {
    c->force_comm = value ? 1 : 0;
    return NGD_OK;
  }
  if (!strcmp(key, "l2u")) {
    c->l2u = value ? 1 : 0;
    c->graph_gen++;
    return NGD_OK;
  }
  if (!strcmp(key, "pdl")) {  // programmatic dependent launch along the PCG kernel chain (process-wide)
    g_pdl = value ? 1 : 0;
    c->graph_gen++;
    return NGD_OK;
  }
  if (!strcmp(key, "l2window")) {
    c->use_l2_window = value ? 1 : 0;
    c->graph_gen++;  // the captured PCG iteration carries the stream's access-policy window
    return NGD_OK;
  }
  if (!strcmp(key, "oz_max_blocks")) {
    if (value < 0 || value > (1 << 30)) return fail(NGD_E_SHAPE, "oz_max_blocks must be >= 0");
    c->oz_max_blocks = (int)value;
    return NGD_OK;
  }
  if (!strcmp(key, "pha_gemm") || !strcmp(key, "out_pre")) {
    // pha_gemm: phase A of the wide layers on the GEMM core (ngd_phag.cu); out_pre: the output
    // layer's Jacobian rows precontracted at linearisation (out_contract); 0 off, 1 on, 2 auto
    if (value < 0 || value > 2) return fail(NGD_E_SHAPE, "%s must be 0, 1 or 2 (auto)", key);
    (key[0] == 'p' ? c->pha_gemm : c->out_pre) = (int)value;
    if (c->have_points) {
      const bool had_out = c->out_on;
      TRY(plan_routes(c));
      // a linearisation made without the precontracted rows cannot serve the new route
      if (c->out_on && !had_out) c->lin_valid = false;
    }
    c->graph_gen++;
    return NGD_OK;
  }
  if (!strcmp(key, "i8_pair")) {
    g_oz_pair = value ? 1 : 0;
    return NGD_OK;
  }
  if (!strcmp(key, "sketch_gemm")) {
    if (value < 0 || value > 2) return fail(NGD_E_SHAPE, "sketch_gemm must be 0 (DMMA), 1 (INT8 Ozaki) or 2 (auto)");
    c->sketch_engine = (int)value;
    return NGD_OK;
  }
  if (!strcmp(key, "svd")) {
    if (value != 1 && value != 3)
      return fail(NGD_E_SHAPE, "svd method must be 1 (cuSOLVER polar SVD) or 3 (FP32 + FP64 block Jacobi, ell <= 512)");
    c->svd_method = (int)value;
    return NGD_OK;
  }
  return fail(NGD_E_SHAPE, "unknown option '%s'", key);
}

int ngd_dot(ngd_ctx* c, const double* x, const double* y, int64_t n, double* h_out) {
  TRY(bind(c));
  dot(x, y, n, c->redp.d(), c->counter(7), c->S(SC_TMP), nullptr, c->stream);
  CK(cudaMemcpyAsync(&c->h_pin[24 + 16], c->S(SC_TMP), sizeof(double), cudaMemcpyDeviceToHost, c->stream));
  CK(cudaStreamSynchronize(c->stream));
  *h_out = c->h_pin[24 + 16];
  return NGD_OK;
}

int ngd_axpy(ngd_ctx* c, const double* a, double alpha, const double* b, double* out, int64_t n) {
  TRY(bind(c));
  theta_minus(a, alpha, b, out, n, c->stream);
  CK(cudaGetLastError());
  return NGD_OK;
}

int ngd_stream_sync(ngd_ctx* c) {
  TRY(bind(c));
  CK(cudaStreamSynchronize(c->stream));
  return NGD_OK;
}

}  // extern "C"
