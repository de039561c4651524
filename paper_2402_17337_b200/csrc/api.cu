// Host runtime and C ABI (include/ibm.h) of the B200 IBM hot path.
//
// One process per GPU.  The grid is split into slabs along y:
// with NCCL (nranks > 1) each process owns one slab and exchanges 2-row halos
// with grouped ncclSend/ncclRecv and the SOR residual with ncclAllReduce(max on
// the uint64 bit pattern, exact); in loopback mode (test) all slabs live in one
// ctx and the same exchanges are device-to-device copies.  Everything stays in
// HBM; per step only the SOR control words and 4 force sums reach the host.
#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstring>
#include <new>
#include <string>

#include <cudaTypedefs.h>
#include <nccl.h>

#include "ibm_internal.h"

using namespace ibm;

struct ibm_ctx : public Ctx {};

namespace {

#define CK(call)                                                                          \
  do {                                                                                    \
    cudaError_t e_ = (call);                                                              \
    if (e_ != cudaSuccess) {                                                              \
      c.err = std::string(#call) + ": " + cudaGetErrorString(e_);                         \
      return IBM_ERR_CUDA;                                                                \
    }                                                                                     \
  } while (0)

#define NK(call)                                                                          \
  do {                                                                                    \
    ncclResult_t r_ = (call);                                                             \
    if (r_ != ncclSuccess) {                                                              \
      c.err = std::string(#call) + ": " + ncclGetErrorString(r_);                         \
      return IBM_ERR_NCCL;                                                                \
    }                                                                                     \
  } while (0)

long round_up(long x, long a) { return (x + a - 1) / a * a; }

struct Carver {
  char *base;
  size_t off;
  template <class T>
  T *take(size_t n) {
    size_t a = (off + 255) & ~size_t(255);
    off = a + n * sizeof(T);
    return base ? reinterpret_cast<T *>(base + a) : nullptr;
  }
};

int check_config(const ibm_config *cfg, std::string &why) {
  if (!cfg) { why = "cfg is NULL"; return IBM_ERR_ARG; }
  if (cfg->nx < 4 || cfg->ny < 4) { why = "nx, ny must be >= 4"; return IBM_ERR_CONFIG; }
  if (!cfg->xn || !cfg->yn) { why = "xn/yn NULL"; return IBM_ERR_ARG; }
  for (int i = 0; i < cfg->nx; ++i)
    if (!(cfg->xn[i + 1] > cfg->xn[i])) { why = "xn not strictly increasing"; return IBM_ERR_CONFIG; }
  for (int j = 0; j < cfg->ny; ++j)
    if (!(cfg->yn[j + 1] > cfg->yn[j])) { why = "yn not strictly increasing"; return IBM_ERR_CONFIG; }
  // spacings within [2^-300, 2^300]: every stencil coefficient and SOR diagonal then
  // lies in [2^-700, 2^700], the range the SOR kernel's division fast path assumes
  for (int i = 0; i < cfg->nx; ++i) {
    const double h = cfg->xn[i + 1] - cfg->xn[i];
    if (!(h >= 0x1p-300 && h <= 0x1p300)) { why = "xn spacing outside [2^-300, 2^300]"; return IBM_ERR_CONFIG; }
  }
  for (int j = 0; j < cfg->ny; ++j) {
    const double h = cfg->yn[j + 1] - cfg->yn[j];
    if (!(h >= 0x1p-300 && h <= 0x1p300)) { why = "yn spacing outside [2^-300, 2^300]"; return IBM_ERR_CONFIG; }
  }
  if (!(cfg->Re > 0)) { why = "Re <= 0"; return IBM_ERR_CONFIG; }
  if (!(cfg->dt > 0)) { why = "dt <= 0"; return IBM_ERR_CONFIG; }
  if (!(cfg->omega_p >= 1.0 && cfg->omega_p < 2.0)) { why = "omega_p outside [1,2)"; return IBM_ERR_CONFIG; }
  if (!(cfg->omega_uv >= 1.0 && cfg->omega_uv < 2.0)) { why = "omega_uv outside [1,2)"; return IBM_ERR_CONFIG; }
  if (!(cfg->tol_p > 0) || !(cfg->tol_uv > 0)) { why = "tolerances must be > 0"; return IBM_ERR_CONFIG; }
  if (cfg->maxit_p < 1 || cfg->maxit_uv < 1) { why = "maxit must be >= 1"; return IBM_ERR_CONFIG; }
  if (cfg->nranks < 1 || (!cfg->loopback && (cfg->rank < 0 || cfg->rank >= cfg->nranks))) {
    why = "rank/nranks inconsistent";
    return IBM_ERR_CONFIG;
  }
  if (cfg->ny / cfg->nranks < 4) { why = "slabs need >= 4 rows"; return IBM_ERR_CONFIG; }
  if (cfg->nranks > 1 && !cfg->loopback && !cfg->nccl_id) { why = "nccl_id required for nranks > 1"; return IBM_ERR_CONFIG; }
  if (cfg->sor_fuse < 0 || cfg->sor_fuse > kWfMaxM) { why = "sor_fuse outside [0, 4]"; return IBM_ERR_CONFIG; }
  return IBM_OK;
}

void slab_rows(int ny, int P, int r, int *j0, int *j1) {
  int base = ny / P, rem = ny % P;
  *j0 = r * base + (r < rem ? r : rem);
  *j1 = *j0 + base + (r < rem ? 1 : 0);
}

// Row pitch in doubles: a multiple of 32 (256 B), plus 32 when that is a multiple
// of 512 (4 KB): power-of-two row strides map the rows a wave of strips reads at
// once onto the same DRAM channels (IBM_PITCH_PAD=0 disables, for measurement).
long row_pitch(int n) {
  long p = round_up(n, 32);
  static const int pad = [] {
    const char *e = std::getenv("IBM_PITCH_PAD");
    return e ? std::atoi(e) : 1;
  }();
  if (pad && p % 512 == 0) p += 32;
  return p;
}

Slab make_slab(const ibm_config &cfg, int r) {
  Slab s;
  std::memset(&s, 0, sizeof(s));
  s.rank = r;
  slab_rows(cfg.ny, cfg.nranks, r, &s.pj0, &s.pj1);
  const int nj = s.pj1 - s.pj0;
  const bool last = (r == cfg.nranks - 1);
  s.gu = Geo{cfg.nx + 1, nj, s.pj0, cfg.ny, row_pitch(cfg.nx + 1)};
  s.gv = Geo{cfg.nx, nj + (last ? 1 : 0), s.pj0, cfg.ny + 1, row_pitch(cfg.nx)};
  s.gp = Geo{cfg.nx, nj, s.pj0, cfg.ny, row_pitch(cfg.nx)};
  s.bu = s.bv = s.bpb = BBox{0, 0, 0, 0};
  return s;
}

size_t rho_len(const ibm_config &cfg) {
  int m = cfg.maxit_p > cfg.maxit_uv ? cfg.maxit_p : cfg.maxit_uv;
  return (size_t)m + 2;
}

// carves everything; base == nullptr -> size only
size_t carve(Ctx &c, char *base) {
  Carver cv{base, 0};
  const int nx = c.cfg.nx, ny = c.cfg.ny;
  Metric &m = c.m;
  m.xn = cv.take<double>(nx + 1); m.yn = cv.take<double>(ny + 1);
  m.dx = cv.take<double>(nx); m.dy = cv.take<double>(ny);
  m.xc = cv.take<double>(nx); m.yc = cv.take<double>(ny);
  m.hxc = cv.take<double>(nx); m.hyc = cv.take<double>(ny);
  m.cEu = cv.take<double>(nx + 1); m.cWu = cv.take<double>(nx + 1); m.cDu = cv.take<double>(nx + 1);
  m.cNu = cv.take<double>(ny); m.cSu = cv.take<double>(ny);
  m.cEv = cv.take<double>(nx); m.cWv = cv.take<double>(nx); m.cDv = cv.take<double>(nx);
  m.cNv = cv.take<double>(ny + 1); m.cSv = cv.take<double>(ny + 1);
  m.cEp = cv.take<double>(nx); m.cWp = cv.take<double>(nx); m.cDp = cv.take<double>(nx);
  m.cNp = cv.take<double>(ny); m.cSp = cv.take<double>(ny);
  c.rho_bits = cv.take<unsigned long long>(rho_len(c.cfg));
  c.ctl = cv.take<SorCtl>(1);
  c.nanflag = cv.take<int>(4);
  for (Slab &s : c.sl) {
    const size_t nu = s.gu.elems(), nv = s.gv.elems(), np = s.gp.elems();
    s.u = cv.take<double>(nu); s.cu = cv.take<double>(nu); s.cup = cv.take<double>(nu);
    s.us[0] = cv.take<double>(nu); s.us[1] = cv.take<double>(nu); s.ru = cv.take<double>(nu);
    s.fu = cv.take<double>(nu);
    s.v = cv.take<double>(nv); s.cv = cv.take<double>(nv); s.cvp = cv.take<double>(nv);
    s.vs[0] = cv.take<double>(nv); s.vs[1] = cv.take<double>(nv); s.rv = cv.take<double>(nv);
    s.fv = cv.take<double>(nv);
    s.p = cv.take<double>(np); s.phi[0] = cv.take<double>(np); s.phi[1] = cv.take<double>(np);
    s.bp = cv.take<double>(np); s.q = cv.take<double>(np);
    s.tu = cv.take<uint8_t>(nu); s.tv = cv.take<uint8_t>(nv); s.tp = cv.take<uint8_t>(np);
    s.pf = cv.take<uint8_t>(np);
    s.red = cv.take<double>(4 + 4 * 64);  // 4 force sums + the per-CTA parts of k_forces_part
  }
  return cv.off + 256;
}

// Host metric arrays: the same formulas as the oracle's, evaluated
// in IEEE double on the host (compiled with -ffp-contract=off).
struct HostMetric {
  std::vector<double> xn, yn, dx, dy, xc, yc, hxc, hyc;
  std::vector<double> cEu, cWu, cDu, cNu, cSu, cEv, cWv, cDv, cNv, cSv, cEp, cWp, cDp, cNp, cSp;
};

HostMetric host_metric(const ibm_config &cfg) {
  const int nx = cfg.nx, ny = cfg.ny;
  HostMetric h;
  h.xn.assign(cfg.xn, cfg.xn + nx + 1);
  h.yn.assign(cfg.yn, cfg.yn + ny + 1);
  h.dx.resize(nx); h.xc.resize(nx); h.hxc.assign(nx, 0.0);
  h.dy.resize(ny); h.yc.resize(ny); h.hyc.assign(ny, 0.0);
  for (int i = 0; i < nx; ++i) { h.dx[i] = h.xn[i + 1] - h.xn[i]; h.xc[i] = 0.5 * (h.xn[i] + h.xn[i + 1]); }
  for (int j = 0; j < ny; ++j) { h.dy[j] = h.yn[j + 1] - h.yn[j]; h.yc[j] = 0.5 * (h.yn[j] + h.yn[j + 1]); }
  for (int i = 1; i < nx; ++i) h.hxc[i] = h.xc[i] - h.xc[i - 1];
  for (int j = 1; j < ny; ++j) h.hyc[j] = h.yc[j] - h.yc[j - 1];
  const auto &dx = h.dx, &dy = h.dy, &hxc = h.hxc, &hyc = h.hyc;
  // u family (interior 1 <= i <= nx-1): zero-gradient outlet, slip walls
  h.cEu.assign(nx + 1, 0.0); h.cWu.assign(nx + 1, 0.0); h.cDu.assign(nx + 1, 0.0);
  h.cNu.assign(ny, 0.0); h.cSu.assign(ny, 0.0);
  for (int i = 1; i <= nx - 1; ++i) {
    if (i <= nx - 2) h.cEu[i] = 1.0 / (hxc[i] * dx[i]);
    h.cWu[i] = 1.0 / (hxc[i] * dx[i - 1]);
  }
  for (int j = 0; j < ny; ++j) {
    if (j <= ny - 2) h.cNu[j] = 1.0 / (dy[j] * hyc[j + 1]);
    if (j >= 1) h.cSu[j] = 1.0 / (dy[j] * hyc[j]);
  }
  // v family (interior 1 <= j <= ny-1): Dirichlet v = 0 on the inlet face, zero-gradient outlet
  h.cEv.assign(nx, 0.0); h.cWv.assign(nx, 0.0); h.cDv.assign(nx, 0.0);
  h.cNv.assign(ny + 1, 0.0); h.cSv.assign(ny + 1, 0.0);
  for (int i = 0; i < nx; ++i) {
    if (i <= nx - 2) h.cEv[i] = 1.0 / (dx[i] * hxc[i + 1]);
    if (i >= 1) h.cWv[i] = 1.0 / (dx[i] * hxc[i]);
  }
  h.cDv[0] = 2.0 / (dx[0] * dx[0]);
  for (int j = 1; j <= ny - 1; ++j) {
    h.cNv[j] = 1.0 / (hyc[j] * dy[j]);
    h.cSv[j] = 1.0 / (hyc[j] * dy[j - 1]);
  }
  // p / phi: Neumann inlet and walls, phi = 0 on the outlet face
  h.cEp.assign(nx, 0.0); h.cWp.assign(nx, 0.0); h.cDp.assign(nx, 0.0);
  h.cNp.assign(ny, 0.0); h.cSp.assign(ny, 0.0);
  for (int i = 0; i < nx; ++i) {
    if (i <= nx - 2) h.cEp[i] = 1.0 / (dx[i] * hxc[i + 1]);
    if (i >= 1) h.cWp[i] = 1.0 / (dx[i] * hxc[i]);
  }
  h.cDp[nx - 1] = 2.0 / (dx[nx - 1] * dx[nx - 1]);
  for (int j = 0; j < ny; ++j) {
    if (j <= ny - 2) h.cNp[j] = 1.0 / (dy[j] * hyc[j + 1]);
    if (j >= 1) h.cSp[j] = 1.0 / (dy[j] * hyc[j]);
  }
  return h;
}

// Eqs. (1)-(2), on the host (same libm as the oracle)
void plunge(double t, double hbar, double k, double *y, double *yd) {
  *y = hbar * sin(k * t);
  *yd = (k * hbar) * cos(k * t);
}

BBox box_for(const std::vector<double> &xs, const std::vector<double> &ys, double xlo, double xhi, double ylo,
             double yhi, const Geo &g, int margin) {
  const int ni = (int)xs.size(), NJ = (int)ys.size();
  int i0 = 0, i1 = ni, j0 = 0, j1 = NJ;
  while (i0 < ni && xs[i0] < xlo) ++i0;
  while (i1 > 0 && xs[i1 - 1] > xhi) --i1;
  while (j0 < NJ && ys[j0] < ylo) ++j0;
  while (j1 > 0 && ys[j1 - 1] > yhi) --j1;
  if (i1 < i0) i1 = i0;
  if (j1 < j0) j1 = j0;
  i0 = std::max(0, i0 - margin); i1 = std::min(ni, i1 + margin);
  j0 = std::max(0, j0 - margin); j1 = std::min(NJ, j1 + margin);
  BBox b{i0, i1, j0 - g.gj0, j1 - g.gj0};
  b.j0 = std::max(b.j0, -kGhost);
  b.j1 = std::min(b.j1, g.nj + kGhost);
  if (b.j1 < b.j0) b.j1 = b.j0;
  return b;
}

// ---------------------------------------------------------------- TMA descriptors
PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  if (!fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  }
  return fn;
}

// 2-D map over a family array incl. its ghost rows: dim0 = columns, dim1 = stored
// rows; elements outside are zero-filled by the TMA unit
bool make_map(CUtensorMap *m, double *base, const Geo &g, int box_h, int box_w = kSorBoxW) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)g.ni, (cuuint64_t)(g.nj + 2 * kGhost)};
  cuuint64_t strides[1] = {(cuuint64_t)g.pitch * sizeof(double)};
  cuuint32_t box[2] = {(cuuint32_t)box_w, (cuuint32_t)box_h};
  cuuint32_t es[2] = {1, 1};
  return fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
            CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_L2_256B,
            CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) == CUDA_SUCCESS;
}

// 1-D coefficient array as a 2-D map of one row (rank-1 maps are rejected by
// the driver on this image); OOB elements are zero-filled
int g_last_encode = 0;
bool make_map_1d(CUtensorMap *m, double *base, int n, int box_n) {
  auto fn = encode_fn();
  if (!fn) return false;
  cuuint64_t dims[2] = {(cuuint64_t)n, 1};
  cuuint64_t strides[1] = {(cuuint64_t)((n * sizeof(double) + 15) / 16 * 16)};
  cuuint32_t box[2] = {(cuuint32_t)box_n, 1};
  cuuint32_t es[2] = {1, 1};
  g_last_encode = (int)fn(m, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, base, dims, strides, box, es,
                          CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
                          CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return g_last_encode == CUDA_SUCCESS;
}

bool make_coef_maps(Ctx &c) {
  const Metric &m = c.m;
  double *arr[3][5] = {{m.cEu, m.cWu, m.cDu, m.cNu, m.cSu},
                       {m.cEv, m.cWv, m.cDv, m.cNv, m.cSv},
                       {m.cEp, m.cWp, m.cDp, m.cNp, m.cSp}};
  const int ncol[3] = {c.nx + 1, c.nx, c.nx}, nrow[3] = {c.ny, c.ny + 1, c.ny};
  for (int f = 0; f < 3; ++f)
    for (int k = 0; k < 5; ++k)
      if (!make_map_1d(&c.tm_coef[f][k], arr[f][k], k < 3 ? ncol[f] : nrow[f], k < 3 ? kSorBoxW : kSorBoxRows1d)) {
        c.err = "cuTensorMapEncodeTiled (coefficients f=" + std::to_string(f) + " k=" + std::to_string(k) +
                " n=" + std::to_string(k < 3 ? ncol[f] : nrow[f]) + " ptr%256=" +
                std::to_string((uintptr_t)arr[f][k] % 256) + " map%64=" + std::to_string((uintptr_t)&c.tm_coef[f][k] % 64) +
                ") -> " + std::to_string(g_last_encode);
        return false;
      }
  return true;
}

bool make_maps(Slab &s, int wf_m) {
  bool ok = true;
  if (wf_m >= 2) {
    ok = ok && make_map(&s.tm_wphi[0], s.phi[0], s.gp, wf_box_rows(wf_m), wf_box_cols());
    ok = ok && make_map(&s.tm_wphi[1], s.phi[1], s.gp, wf_box_rows(wf_m), wf_box_cols());
    ok = ok && make_map(&s.tm_wbp, s.bp, s.gp, wf_box_rows(wf_m), wf_box_cols());
  }
  for (int q = 0; q < 2; ++q) {
    ok = ok && make_map(&s.tm_phi[q], s.phi[q], s.gp, kSorBoxHx);
    ok = ok && make_map(&s.tm_us[q], s.us[q], s.gu, kSorBoxHx);
    ok = ok && make_map(&s.tm_vs[q], s.vs[q], s.gv, kSorBoxHx);
  }
  ok = ok && make_map(&s.tm_bp, s.bp, s.gp, kSorBoxHb);
  ok = ok && make_map(&s.tm_ru, s.ru, s.gu, kSorBoxHb);
  ok = ok && make_map(&s.tm_rv, s.rv, s.gv, kSorBoxHb);
  return ok;
}

// ---------------------------------------------------------------- halos and reductions
// exchange 2 ghost rows of one family buffer (selected per slab by `pick`)
template <class Pick>
int halo(Ctx &c, Pick pick, int rows = 2, cudaStream_t st = nullptr, bool on_comm = false) {
  const size_t esz = sizeof(double);
  if (!on_comm) st = c.stream;
  if (c.loopback) {
    for (size_t r = 0; r + 1 < c.sl.size(); ++r) {
      double *lo, *up;
      const Geo *glo, *gup;
      pick(c.sl[r], &lo, &glo);
      pick(c.sl[r + 1], &up, &gup);
      const size_t bytes = (size_t)rows * glo->pitch * esz;
      CK(cudaMemcpyAsync(up + gup->off(0, -rows), lo + glo->off(0, glo->nj - rows), bytes,
                         cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(lo + glo->off(0, glo->nj), up + gup->off(0, 0), bytes, cudaMemcpyDeviceToDevice, st));
    }
    return IBM_OK;
  }
  if (c.nranks == 1) return IBM_OK;
  // (the overlapped exchanges use their own communicator: NCCL operations of one
  // communicator must not run concurrently on two streams)
  ncclComm_t comm = (ncclComm_t)(on_comm ? c.nccl_halo : c.nccl);
  double *buf;
  const Geo *g;
  pick(c.sl[0], &buf, &g);
  const int r = c.sl[0].rank;
  const size_t cnt = (size_t)rows * g->pitch;
  NK(ncclGroupStart());
  if (r > 0) {
    NK(ncclSend(buf + g->off(0, 0), cnt, ncclFloat64, r - 1, comm, st));
    NK(ncclRecv(buf + g->off(0, -rows), cnt, ncclFloat64, r - 1, comm, st));
  }
  if (r < c.nranks - 1) {
    NK(ncclSend(buf + g->off(0, g->nj - rows), cnt, ncclFloat64, r + 1, comm, st));
    NK(ncclRecv(buf + g->off(0, g->nj), cnt, ncclFloat64, r + 1, comm, st));
  }
  NK(ncclGroupEnd());
  return IBM_OK;
}

#define HALO(expr)                                                            \
  do {                                                                        \
    int st_ = halo(c, [&](Slab &s, double **b, const Geo **g) { expr; });     \
    if (st_) return st_;                                                      \
  } while (0)
// the same with `rows` ghost rows (the fused Poisson pass needs 2m)
#define HALO_ROWS(rows, expr)                                                   \
  do {                                                                          \
    int st_ = halo(c, [&](Slab &s, double **b, const Geo **g) { expr; }, rows); \
    if (st_) return st_;                                                        \
  } while (0)
// ... on the comm stream with the halo communicator (overlapped with the pass)
#define HALO_ROWS_COMM(rows, expr)                                                              \
  do {                                                                                          \
    int st_ = halo(c, [&](Slab &s, double **b, const Geo **g) { expr; }, rows, c.comm, true);   \
    if (st_) return st_;                                                                        \
  } while (0)

bool multi(const Ctx &c) { return c.sl.size() > 1 || c.nranks > 1; }

// Sums of the 4 force partials over slabs (loopback: host, in slab order) or
// ranks (NCCL sum all-reduce, in place, before the copy).
int force_sums(Ctx &c, double out[4]) {
  if (!c.loopback && c.nranks > 1) {
    NK(ncclAllReduce(c.sl[0].red, c.sl[0].red, 4, ncclFloat64, ncclSum, (ncclComm_t)c.nccl, c.stream));
    NK(ncclAllReduce(c.nanflag, c.nanflag, 1, ncclInt32, ncclMax, (ncclComm_t)c.nccl, c.stream));
  }
  for (size_t r = 0; r < c.sl.size(); ++r)
    CK(cudaMemcpyAsync(c.h_red + 4 * r, c.sl[r].red, 4 * sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaMemcpyAsync(c.h_nan, c.nanflag, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  for (int q = 0; q < 4; ++q) out[q] = 0.0;
  for (size_t r = 0; r < c.sl.size(); ++r)
    for (int q = 0; q < 4; ++q) out[q] = out[q] + c.h_red[4 * r + q];
  return IBM_OK;
}

// solid momentum M at the current tags and fields (R20)
int refresh_time(Ctx &c) {
  const double t = (double)c.step * c.cfg.dt;
  double yb = c.body.y0, vb = 0.0, disp = 0.0;
  if (c.body.has) {
    plunge(t, c.body.hbar, c.body.k, &disp, &vb);
    yb = c.body.y0 + disp;
    for (Slab &s : c.sl) launch_classify(c, s, yb);
  }
  for (Slab &s : c.sl) launch_forces(c, s);
  CK(cudaGetLastError());
  double sums[4];
  int st = force_sums(c, sums);
  if (st) return st;
  c.Mx = sums[1];
  c.My = sums[3];
  return IBM_OK;
}

// ---------------------------------------------------------------- SOR driver
// Launches iterations in batches; each iteration kernel early-exits once the
// device control block says converged, so the host polls once per batch.
// One SOR solve from the iterate in buffer s0.  Passes are launched in
// batches between convergence polls; a pass is one iteration (k_sor) or, for the
// single-slab Poisson system, wf_m fused iterations (k_sor_wf).  The pass's last
// CTA takes the convergence decision on the device; if it stops at an iteration
// inside a fused pass, that pass is replayed from its (intact) input buffer up to
// the decided iteration.  *buf_out receives the buffer index of the result.
// IBM_DEBUG_SYNC=1: synchronise and check after every phase of a step (locates a
// faulting kernel; debugging only)
static bool debug_sync() {
  static const bool on = [] {
    const char *e = std::getenv("IBM_DEBUG_SYNC");
    return e && std::atoi(e) == 1;
  }();
  return on;
}
#define DSYNC(tag)                                                                    \
  do {                                                                                \
    if (debug_sync()) {                                                               \
      cudaError_t e_ = cudaStreamSynchronize(c.stream);                               \
      if (e_ != cudaSuccess) {                                                        \
        c.err = std::string("after ") + (tag) + ": " + cudaGetErrorString(e_);        \
        return IBM_ERR_CUDA;                                                          \
      }                                                                               \
    }                                                                                 \
  } while (0)

// The fused pass's per-segment table (WfSeg) for slab r at the plan's segment
// length: built on the host from the row coefficients once per (slab, L) and
// uploaded on the solver stream; kept until ibm_destroy.
int wf_attach_seg(Ctx &c, size_t r, WfArgs &wa) {
  const long key = (long)r * 1000000L + wa.L;
  auto it = c.wf_segs.find(key);
  if (it == c.wf_segs.end()) {
    std::vector<WfSeg> tab = wf_seg_table(wa, c.wf_m, c.h_cNp.data(), c.h_cSp.data());
    WfSeg *d = nullptr;
    if (cudaMalloc(&d, tab.size() * sizeof(WfSeg)) != cudaSuccess) {
      c.err = "cudaMalloc (fused-pass segment table)";
      return IBM_ERR_CUDA;
    }
    it = c.wf_segs.emplace(key, std::make_pair(std::move(tab), d)).first;
    if (cudaMemcpyAsync(d, it->second.first.data(), it->second.first.size() * sizeof(WfSeg),
                        cudaMemcpyHostToDevice, c.stream) != cudaSuccess) {
      c.err = "cudaMemcpyAsync (fused-pass segment table)";
      return IBM_ERR_CUDA;
    }
  }
  wa.seg = it->second.second;
  return IBM_OK;
}

int sor_solve(Ctx &c, bool helm, int s0, int *k_out, double *rho_out, int *status, int iters_override,
              int *buf_out) {
  const ibm_config &cfg = c.cfg;
  const int maxit = iters_override > 0 ? iters_override : (helm ? cfg.maxit_uv : cfg.maxit_p);
  const double tol = iters_override > 0 ? -1.0 : (helm ? cfg.tol_uv : cfg.tol_p);
  const double omega = helm ? cfg.omega_uv : cfg.omega_p;
  CK(cudaMemsetAsync(c.rho_bits, 0, sizeof(unsigned long long) * (size_t)(maxit + 2), c.stream));
  std::memset(&c.h_ctl[1], 0, sizeof(SorCtl));
  c.h_ctl[1].k_done = -1;
  CK(cudaMemcpyAsync(c.ctl, &c.h_ctl[1], sizeof(SorCtl), cudaMemcpyHostToDevice, c.stream));
  const bool mult = multi(c);
  std::vector<SorArgs> args(c.sl.size());
  std::vector<int> grids(c.sl.size());
  for (size_t r = 0; r < c.sl.size(); ++r) {
    Slab &s = c.sl[r];
    SorArgs &a = args[r];
    std::memset(&a, 0, sizeof(a));
    a.helmholtz = helm ? 1 : 0;
    a.beta = cfg.dt * (0.5 / cfg.Re);
    a.omega = omega;
    a.omc = 1.0 - omega;
    a.tol = tol;
    a.maxit = maxit;
    a.check_every = cfg.check_every;
    a.rho_bits = c.rho_bits;
    a.ctl = c.ctl;
    a.multi = mult ? 1 : 0;
    auto fam = [&](SorFam &f, const Geo &g, const double *b, const uint8_t *flag, const BBox &box,
                   const double *cE, const double *cW, const double *cD, const double *cN, const double *cS, int ui0,
                   int ui1, int uj0, int uj1, int fid) {
      f.g = g; f.b = b; f.flag = flag; f.box = box;
      for (int k = 0; k < 5; ++k) f.tmc[k] = c.tm_coef[fid][k];
      f.cE = cE; f.cW = cW; f.cD = cD; f.cN = cN; f.cS = cS;
      f.ui0 = ui0; f.ui1 = ui1; f.uj0 = uj0; f.uj1 = uj1;
      f.tiles_x = (g.ni + kSorTileX - 1) / kSorTileX;
      f.tiles_y = (g.nj + kSorTileY - 1) / kSorTileY;
    };
    const Metric &m = c.m;
    if (helm) {
      fam(a.f[0], s.gu, s.ru, s.tu, s.bu, m.cEu, m.cWu, m.cDu, m.cNu, m.cSu, 1, c.nx, 0, c.ny, 0);
      fam(a.f[1], s.gv, s.rv, s.tv, s.bv, m.cEv, m.cWv, m.cDv, m.cNv, m.cSv, 0, c.nx, 1, c.ny, 1);
      a.nfam = 2;
    } else {
      BBox pb = s.bpb;
      fam(a.f[0], s.gp, s.bp, s.pf, pb, m.cEp, m.cWp, m.cDp, m.cNp, m.cSp, 0, c.nx, 0, c.ny, 2);
      a.nfam = 1;
    }
    a.total_tiles = a.f[0].tiles_x * a.f[0].tiles_y + (a.nfam == 2 ? a.f[1].tiles_x * a.f[1].tiles_y : 0);
    grids[r] = sor_grid(a);
  }
  if (!helm && !mult && c.tb_m >= 2 && cfg.sor_batch <= 0) {
    // mid-size grid: the resident, temporally blocked persistent solve (sor_tb.cu)
    TbArgs a = c.tb;
    Slab &s = c.sl[0];
    a.xb[0] = s.phi[0];
    a.xb[1] = s.phi[1];
    a.b = s.bp;
    a.flag = s.pf;
    a.box = s.bpb;
    a.s0 = s0;
    a.omega = omega;
    a.tol = tol;
    a.maxit = maxit;
    a.check_every = cfg.check_every;
    a.rho_bits = c.rho_bits;
    a.ctl = c.ctl;
    CK(launch_sor_tb(a, c.stream));
    ++c.launches;
    CK(cudaMemcpyAsync(&c.h_ctl[0], c.ctl, sizeof(SorCtl), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    *k_out = c.h_ctl[0].k_done;
    unsigned long long rb = c.h_ctl[0].rho_final;
    std::memcpy(rho_out, &rb, sizeof(double));
    *status = c.h_ctl[0].status;
    *buf_out = c.h_ctl[0].buf;
    if (iters_override <= 0) c.hint_p = *k_out;
    return IBM_OK;
  }
  if (!mult && iters_override <= 0 && cfg.sor_batch <= 0 && sor_coop_fits(args[0])) {
    // small grid: the whole loop in one persistent cooperative launch
    Slab &s = c.sl[0];
    SorArgs &a = args[0];
    if (helm) {
      a.f[0].xb[0] = s.us[0]; a.f[0].xb[1] = s.us[1]; a.f[0].tmxb[0] = s.tm_us[0]; a.f[0].tmxb[1] = s.tm_us[1];
      a.f[0].tmb = s.tm_ru;
      a.f[1].xb[0] = s.vs[0]; a.f[1].xb[1] = s.vs[1]; a.f[1].tmxb[0] = s.tm_vs[0]; a.f[1].tmxb[1] = s.tm_vs[1];
      a.f[1].tmb = s.tm_rv;
    } else {
      a.f[0].xb[0] = s.phi[0]; a.f[0].xb[1] = s.phi[1]; a.f[0].tmxb[0] = s.tm_phi[0]; a.f[0].tmxb[1] = s.tm_phi[1];
      a.f[0].tmb = s.tm_bp;
    }
    CK(launch_sor_coop(a, s0, c.stream));
    ++c.launches;
    CK(cudaMemcpyAsync(&c.h_ctl[0], c.ctl, sizeof(SorCtl), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    *k_out = c.h_ctl[0].k_done;
    unsigned long long rb = c.h_ctl[0].rho_final;
    std::memcpy(rho_out, &rb, sizeof(double));
    *status = c.h_ctl[0].status;
    *buf_out = (s0 + *k_out) & 1;
    return IBM_OK;
  }
  // temporally blocked Poisson passes (every slab; decomposed runs exchange 2m
  // halo rows per pass and reduce the m residuals after it)
  const bool wf = !helm && c.wf_m >= 2;
  std::vector<WfArgs> was(wf ? c.sl.size() : 0);
  for (size_t r = 0; r < was.size(); ++r) {
    WfArgs &wa = was[r];
    std::memset(&wa, 0, sizeof(wa));
    const Slab &s = c.sl[r];
    const SorFam &f = args[r].f[0];
    wa.tmb = s.tm_wbp;
    wa.flag = f.flag; wa.g = f.g; wa.box = f.box;
    wa.cE = f.cE; wa.cW = f.cW; wa.cD = f.cD; wa.cN = f.cN; wa.cS = f.cS;
    wa.ui0 = f.ui0; wa.ui1 = f.ui1; wa.uj0 = f.uj0; wa.uj1 = f.uj1;
    wa.omega = omega; wa.omc = 1.0 - omega; wa.tol = tol;
    wa.maxit = maxit; wa.check_every = cfg.check_every;
    wa.rho_bits = c.rho_bits; wa.ctl = c.ctl;
    wa.multi = mult ? 1 : 0;
    wf_plan(wa, c.wf_m);
    if (int e = wf_attach_seg(c, r, wa)) return e;
  }
  // decomposed fused passes: an exchange of the last pass's output may be in
  // flight on the comm stream; the main stream joins it before touching ghost rows
  bool halo_ready = false;
  bool peer_ready = false;  // ghost rows of buffer `cur` hold the neighbours' rows (peer-halo passes)
  auto join_comm = [&]() -> int {
    if (halo_ready) CK(cudaStreamWaitEvent(c.stream, c.ev_halo, 0));
    halo_ready = false;
    return IBM_OK;
  };
  // one single-iteration pass of every slab (halos first when decomposed)
  auto single = [&](int kk, int in, bool fixup) -> int {
    const int out = in ^ 1;
    peer_ready = false;  // (its output's ghost rows are not written)
    if (mult) {
      if (int e = join_comm()) return e;
      if (helm) {
        HALO((*b = s.us[in], *g = &s.gu));
        HALO((*b = s.vs[in], *g = &s.gv));
      } else {
        HALO((*b = s.phi[in], *g = &s.gp));
      }
    }
    for (size_t r = 0; r < c.sl.size(); ++r) {
      Slab &s = c.sl[r];
      SorArgs &a = args[r];
      a.k = kk;
      a.fixup = fixup ? 1 : 0;
      if (helm) {
        a.f[0].xin = s.us[in]; a.f[0].xout = s.us[out]; a.f[0].tmx = s.tm_us[in]; a.f[0].tmb = s.tm_ru;
        a.f[1].xin = s.vs[in]; a.f[1].xout = s.vs[out]; a.f[1].tmx = s.tm_vs[in]; a.f[1].tmb = s.tm_rv;
      } else {
        a.f[0].xin = s.phi[in]; a.f[0].xout = s.phi[out]; a.f[0].tmx = s.tm_phi[in]; a.f[0].tmb = s.tm_bp;
      }
      DSYNC("sor halo / previous pass");
      launch_sor_iteration(a, c.stream, grids[r]);
      ++c.launches;
      DSYNC(helm ? "k_sor<1> iteration" : "k_sor<0> iteration");
    }
    if (mult && !fixup) {
      if (!c.loopback)
        NK(ncclAllReduce(c.rho_bits + kk, c.rho_bits + kk, 1, ncclUint64, ncclMax, (ncclComm_t)c.nccl, c.stream));
      launch_sor_check(c.ctl, c.rho_bits, kk, maxit, cfg.check_every, tol, c.stream);
      ++c.launches;
    }
    return IBM_OK;
  };
  struct Pass {
    int k0, m, in;
  };
  std::vector<Pass> passes;
  int &hint = helm ? c.hint_uv : c.hint_p;
  int batch = cfg.sor_batch > 0 ? cfg.sor_batch : std::max(4, std::min(hint, maxit));
  int k = 1, cur = s0;
  // Online tuning of the fused pass's segment length (single slab, no
  // IBM_WF_ROWS): the first 2 x ncand fused passes of a run cycle through the
  // candidates (wf_candidates), each timed by its own events; the fastest is kept
  // for the rest of the run.  Every length gives the same iterates, so these are
  // ordinary passes of the solve.
  std::vector<int> cand;
  int tune_n = 0, tune_launched = 0, tune_k_end = 0;
  if (wf && !mult) {
    if (c.wf_L == 0 && !std::getenv("IBM_WF_ROWS")) {
      cand = wf_candidates(c.sl[0].gp, c.wf_m);
      if (cand.size() > 1)
        tune_n = std::min(2 * (int)cand.size(), 12);  // each candidate twice
      else
        c.wf_L = cand[0];
    }
    if (c.wf_L > 0) {
      wf_plan(was[0], c.wf_m, c.wf_L);
      if (int e = wf_attach_seg(c, 0, was[0])) return e;
    }
  }
  for (;;) {
    const int kend = std::min(maxit, k + batch - 1);
    while (k <= kend) {
      if (wf && mult && c.peer_halo && k + c.wf_m - 1 <= maxit) {
        // Decomposed grid, device-initiated halo (f3): each slab's pass also stores its
        // 2m boundary rows of output straight into the neighbours' ghost rows of their
        // next input buffer (loopback: the other slabs' buffers; ranks: CUDA-IPC
        // mappings over NVLink).  The per-pass residual all-reduce orders those
        // stores before any rank's next pass (each rank contributes only after its
        // pass kernel completed), so no further exchange or flag is needed.  The
        // first pass of a solve, and the first after one-iteration passes, exchanges
        // its input's ghost rows once.
        const int in = cur;
        if (!peer_ready) HALO_ROWS(2 * c.wf_m, (*b = s.phi[in], *g = &s.gp));
        for (size_t r = 0; r < c.sl.size(); ++r) {
          WfArgs wa = was[r];
          wa.k = k;
          wa.xout = c.sl[r].phi[in ^ 1];
          wa.tmx = c.sl[r].tm_wphi[in];
          wa.peer_rows = 2 * c.wf_m;
          const long pitch = c.sl[r].gp.pitch;
          if (c.loopback) {
            wa.peer_lo = r > 0 ? c.sl[r - 1].phi[in ^ 1] + (long)c.sl[r - 1].gp.nj * pitch : nullptr;
            wa.peer_hi = r + 1 < c.sl.size() ? c.sl[r + 1].phi[in ^ 1] - (long)c.sl[r].gp.nj * pitch : nullptr;
          } else {
            wa.peer_lo = c.peer_phi[0][in ^ 1] ? c.peer_phi[0][in ^ 1] + (long)c.peer_nj[0] * pitch : nullptr;
            wa.peer_hi = c.peer_phi[1][in ^ 1] ? c.peer_phi[1][in ^ 1] - (long)c.sl[r].gp.nj * pitch : nullptr;
          }
          CK(launch_sor_wf(wa, c.wf_m, c.stream));
          ++c.launches;
        }
        if (!c.loopback)
          NK(ncclAllReduce(c.rho_bits + k, c.rho_bits + k, c.wf_m, ncclUint64, ncclMax, (ncclComm_t)c.nccl,
                           c.stream));
        launch_sor_check(c.ctl, c.rho_bits, k, maxit, cfg.check_every, tol, c.stream, c.wf_m, wf_approx() ? 1 : 0);
        ++c.launches;
        passes.push_back({k, c.wf_m, cur});
        k += c.wf_m;
        peer_ready = true;
      } else if (wf && mult && k + c.wf_m - 1 <= maxit) {
        // Decomposed grid: the 2m halo rows of this pass's input arrived on the comm
        // stream (the first pass: exchanged here); the edge segments (those that read
        // ghost rows) run first, then the interior ones while the comm stream already
        // exchanges the edge rows of this pass's output for the next pass.
        const int in = cur;
        if (!halo_ready) HALO_ROWS(2 * c.wf_m, (*b = s.phi[in], *g = &s.gp));
        else CK(cudaStreamWaitEvent(c.stream, c.ev_halo, 0));
        for (int mode = 1; mode <= 2; ++mode) {
          for (size_t r = 0; r < c.sl.size(); ++r) {
            WfArgs wa = was[r];
            const int nseg = mode == 1 ? wa.e_lo + wa.e_hi : wa.segs - wa.e_lo - wa.e_hi;
            if (nseg <= 0) continue;
            wa.seg_mode = mode;
            wa.items = wa.strips * nseg;
            wa.k = k;
            wa.xout = c.sl[r].phi[in ^ 1];
            wa.tmx = c.sl[r].tm_wphi[in];
            CK(launch_sor_wf(wa, c.wf_m, c.stream));
            ++c.launches;
          }
          if (mode == 1) {
            CK(cudaEventRecord(c.ev_edge, c.stream));
            CK(cudaStreamWaitEvent(c.comm, c.ev_edge, 0));
            HALO_ROWS_COMM(2 * c.wf_m, (*b = s.phi[in ^ 1], *g = &s.gp));
            CK(cudaEventRecord(c.ev_halo, c.comm));
            halo_ready = true;
          }
        }
        if (!c.loopback)
          NK(ncclAllReduce(c.rho_bits + k, c.rho_bits + k, c.wf_m, ncclUint64, ncclMax, (ncclComm_t)c.nccl,
                           c.stream));
        launch_sor_check(c.ctl, c.rho_bits, k, maxit, cfg.check_every, tol, c.stream, c.wf_m, wf_approx() ? 1 : 0);
        ++c.launches;
        passes.push_back({k, c.wf_m, cur});
        k += c.wf_m;
      } else if (wf && k + c.wf_m - 1 <= maxit) {
        const int in = cur;
        const bool tuning = tune_launched < tune_n;
        if (tuning) {
          wf_plan(was[0], c.wf_m, cand[tune_launched % cand.size()]);
          if (int e = wf_attach_seg(c, 0, was[0])) return e;
          CK(cudaEventRecord(c.tev[2 * tune_launched], c.stream));
        }
        for (size_t r = 0; r < c.sl.size(); ++r) {
          WfArgs &wa = was[r];
          wa.k = k;
          wa.xout = c.sl[r].phi[in ^ 1];
          wa.tmx = c.sl[r].tm_wphi[in];
          CK(launch_sor_wf(wa, c.wf_m, c.stream));
          ++c.launches;
        }
        if (tuning) {
          CK(cudaEventRecord(c.tev[2 * tune_launched + 1], c.stream));
          if (++tune_launched == tune_n) tune_k_end = k + c.wf_m - 1;
        }
        // the decision of every fused pass: first of its m iterations that may stop
        launch_sor_check(c.ctl, c.rho_bits, k, maxit, cfg.check_every, tol, c.stream, c.wf_m, wf_approx() ? 1 : 0);
        ++c.launches;
        passes.push_back({k, c.wf_m, cur});
        k += c.wf_m;
      } else {
        int r = single(k, cur, false);
        if (r) return r;
        passes.push_back({k, 1, cur});
        k += 1;
      }
      cur ^= 1;
    }
    CK(cudaGetLastError());
    CK(cudaMemcpyAsync(&c.h_ctl[0], c.ctl, sizeof(SorCtl), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    if (tune_n > 0 && tune_launched == tune_n && c.wf_L == 0) {
      // all tuning passes ran in full unless the solve stopped inside them (then
      // the next run tunes again)
      if (c.h_ctl[0].k_done < 0 || c.h_ctl[0].k_done >= tune_k_end) {
        std::vector<float> best(cand.size(), 1e30f);
        for (int i = 0; i < tune_n; ++i) {
          float ms = 0.f;
          if (cudaEventElapsedTime(&ms, c.tev[2 * i], c.tev[2 * i + 1]) == cudaSuccess)
            best[i % cand.size()] = std::min(best[i % cand.size()], ms);
        }
        c.wf_L = cand[std::min_element(best.begin(), best.end()) - best.begin()];
        wf_plan(was[0], c.wf_m, c.wf_L);
        if (int e = wf_attach_seg(c, 0, was[0])) return e;
      }
      tune_n = 0;
    }
    if (c.h_ctl[0].k_done >= 0 && c.h_ctl[0].status == 4) {
      // Provisional stop in a fused pass with the approximate (high-word) residual:
      // replay that pass from its intact input with exact one-iteration passes --
      // the same iterates, exact residuals, exact device-side decision.
      const int kp = c.h_ctl[0].k_done;
      size_t pi = 0;
      while (pi < passes.size() && !(kp >= passes[pi].k0 && kp < passes[pi].k0 + passes[pi].m)) ++pi;
      if (pi == passes.size()) { c.err = "provisional SOR stop at an iteration no pass covers"; return IBM_ERR_STATE; }
      const Pass P = passes[pi];
      passes.resize(pi);
      std::memset(&c.h_ctl[1], 0, sizeof(SorCtl));
      c.h_ctl[1].k_done = -1;
      CK(cudaMemcpyAsync(c.ctl, &c.h_ctl[1], sizeof(SorCtl), cudaMemcpyHostToDevice, c.stream));
      int in = P.in;
      for (int kk = P.k0; kk < P.k0 + P.m; ++kk, in ^= 1) {
        int r = single(kk, in, false);
        if (r) return r;
        passes.push_back({kk, 1, in});
      }
      k = P.k0 + P.m;
      cur = in;
      CK(cudaMemcpyAsync(&c.h_ctl[0], c.ctl, sizeof(SorCtl), cudaMemcpyDeviceToHost, c.stream));
      CK(cudaStreamSynchronize(c.stream));
      if (c.h_ctl[0].k_done >= 0) break;  // exact stop inside the replayed pass
      continue;                            // the bound was not tight: carry on after the pass
    }
    if (c.h_ctl[0].k_done >= 0) break;
    if (cfg.sor_batch <= 0) batch = std::min(2 * batch, 1024);
  }
  const int kd = c.h_ctl[0].k_done;
  *k_out = kd;
  unsigned long long rb = c.h_ctl[0].rho_final;
  std::memcpy(rho_out, &rb, sizeof(double));
  *status = c.h_ctl[0].status;
  // the pass that holds iteration kd; replay a fused pass that overshot it
  int buf = -1;
  for (const Pass &p : passes)
    if (kd >= p.k0 && kd < p.k0 + p.m) {
      buf = p.in ^ 1;
      if (kd < p.k0 + p.m - 1) {
        int in = p.in;
        for (int kk = p.k0; kk <= kd; ++kk, in ^= 1) {
          int r = single(kk, in, true);
          if (r) return r;
        }
        buf = in;
      }
      break;
    }
  if (buf < 0) { c.err = "SOR stopped at an iteration no pass covers"; return IBM_ERR_STATE; }
  if (int e = join_comm()) return e;
  *buf_out = buf;
  if (iters_override <= 0) hint = *k_out;
  return IBM_OK;
}

float ev_ms(Ctx &c, int a, int b) {
  float ms = 0.f;
  if (cudaEventElapsedTime(&ms, c.ev[a], c.ev[b]) != cudaSuccess) ms = 0.f;
  return ms;
}

// ---------------------------------------------------------------- one step n -> n+1
int step_once(Ctx &c, ibm_step_stats *st) {
  const double dt = c.cfg.dt;
  const double t1 = (double)(c.step + 1) * dt;  // R13: not accumulated
  double disp = 0.0, vb = 0.0;
  if (c.body.has) plunge(t1, c.body.hbar, c.body.k, &disp, &vb);
  const double yb = c.body.y0 + disp;
  int status = IBM_OK;
  c.launches = 0;
  CK(cudaEventRecord(c.ev[0], c.stream));
  // a1 classification at t^{n+1} (R15) + Poisson masks
  if (c.body.has)
    for (Slab &s : c.sl) {
      c.launches += launch_classify(c, s, yb);
      DSYNC("classify");
      c.launches += launch_pflags(c, s);
      DSYNC("pflags");
    }
  CK(cudaEventRecord(c.ev[7], c.stream));
  // N1 halos of u^n, v^n, p^n, then a2/a3 predictor
  if (multi(c)) {
    HALO((*b = s.u, *g = &s.gu));
    HALO((*b = s.v, *g = &s.gv));
    HALO((*b = s.p, *g = &s.gp));
  }
  DSYNC("halo u v p");
  for (Slab &s : c.sl) c.launches += launch_predictor(c, s, yb, vb);
  CK(cudaGetLastError());
  DSYNC("predictor");
  // the fused red-black pass also updates red on the first ghost row: it needs
  // the neighbour's right-hand side there
  if (multi(c)) {
    HALO((*b = s.ru, *g = &s.gu));
    HALO((*b = s.rv, *g = &s.gv));
  }
  CK(cudaEventRecord(c.ev[1], c.stream));
  DSYNC("halo rhs");
  // a4 velocity (Helmholtz) SOR, u and v jointly (R5)
  int ku = 0, sst = 0;
  double rho_uv = 0.0;
  int ures = 0;
  int r = sor_solve(c, true, 0, &ku, &rho_uv, &sst, 0, &ures);
  if (r) return r;
  if (st) { st->it_uv = ku; st->rho_uv = rho_uv; }
  DSYNC("velocity SOR");
  if (sst == 3) { c.err = "velocity SOR residual is NaN at step " + std::to_string(c.step + 1); return IBM_ERR_DIVERGED; }
  if (sst == 1) status = IBM_WARN_NOCONV;
  // the outlet fill (R10b) reads v* one row up: exchange v* first, then u*
  if (multi(c)) HALO((*b = s.vs[ures], *g = &s.gv));
  for (Slab &s : c.sl) c.launches += launch_outlet_fill(c, s, s.us[ures], s.vs[ures]);
  if (multi(c)) HALO((*b = s.us[ures], *g = &s.gu));
  CK(cudaEventRecord(c.ev[2], c.stream));
  DSYNC("outlet fill + halos");
  // a5 masks -> q, Poisson rhs; phi := 0 on inactive cells
  for (Slab &s : c.sl) c.launches += launch_prhs(c, s, s.us[ures], s.vs[ures], s.phi[c.phi_cur]);
  if (multi(c)) HALO_ROWS(c.wf_m >= 2 ? 2 * c.wf_m : 2, (*b = s.bp, *g = &s.gp));
  CK(cudaEventRecord(c.ev[3], c.stream));
  DSYNC("poisson rhs");
  // a6 Poisson SOR, warm start
  int kp = 0;
  double rho_p = 0.0;
  int pbuf = c.phi_cur;
  r = sor_solve(c, false, c.phi_cur, &kp, &rho_p, &sst, 0, &pbuf);
  if (r) return r;
  if (st) { st->it_p = kp; st->rho_p = rho_p; }
  DSYNC("poisson SOR");
  if (sst == 3) { c.err = "pressure SOR residual is NaN at step " + std::to_string(c.step + 1); return IBM_ERR_DIVERGED; }
  if (sst == 1) status = IBM_WARN_NOCONV;
  c.phi_cur = pbuf;
  if (multi(c)) HALO((*b = s.phi[c.phi_cur], *g = &s.gp));
  CK(cudaEventRecord(c.ev[4], c.stream));
  // a7 projection
  CK(cudaMemsetAsync(c.nanflag, 0, sizeof(int), c.stream));
  for (Slab &s : c.sl) c.launches += launch_correct(c, s, s.us[ures], s.vs[ures], s.phi[c.phi_cur]);
  if (c.body.has)
    for (Slab &s : c.sl) c.launches += launch_pext(c, s, s.phi[c.phi_cur]);
  CK(cudaEventRecord(c.ev[5], c.stream));
  DSYNC("correct");
  // history rotation
  for (Slab &s : c.sl) {
    std::swap(s.cu, s.cup);
    std::swap(s.cv, s.cvp);
  }
  c.have_hist = 1;
  // a8 forces
  for (Slab &s : c.sl) c.launches += launch_forces(c, s);
  CK(cudaGetLastError());
  CK(cudaEventRecord(c.ev[6], c.stream));
  double sums[4];
  r = force_sums(c, sums);
  if (r) return r;
  const double Fx = -sums[0] + (sums[1] - c.Mx) / dt;
  const double Fy = -sums[2] + (sums[3] - c.My) / dt;
  c.Mx = sums[1];
  c.My = sums[3];
  c.last_t = t1;
  c.last_cd = 2.0 * Fx;
  c.last_cl = 2.0 * Fy;
  c.step += 1;
  if (st) {
    st->step = c.step;
    st->t_bar = t1;
    st->cd = c.last_cd;
    st->cl = c.last_cl;
    st->ms[0] = ev_ms(c, 0, 1);
    st->ms[1] = ev_ms(c, 1, 2);
    st->ms[2] = ev_ms(c, 2, 3);
    st->ms[3] = ev_ms(c, 3, 4);
    st->ms[4] = ev_ms(c, 4, 5);
    st->ms[5] = ev_ms(c, 5, 6);
    st->ms[6] = ev_ms(c, 0, 7);
    st->ms[7] = ev_ms(c, 0, 6);
    st->launches = c.launches;
  }
  if (*c.h_nan) {
    c.err = "non-finite field after correction at step " + std::to_string(c.step);
    return IBM_ERR_DIVERGED;
  }
  return status;
}

const char *kNoCtx = "ctx is NULL";

}  // namespace

// ================================================================ C ABI
extern "C" {

int ibm_workspace_size(const ibm_config *cfg, size_t *bytes) {
  std::string why;
  int st = check_config(cfg, why);
  if (st) return st;
  if (!bytes) return IBM_ERR_ARG;
  Ctx c;
  c.cfg = *cfg;
  c.loopback = cfg->loopback;
  if (cfg->loopback)
    for (int r = 0; r < cfg->nranks; ++r) c.sl.push_back(make_slab(*cfg, r));
  else
    c.sl.push_back(make_slab(*cfg, cfg->rank));
  *bytes = carve(c, nullptr);
  return IBM_OK;
}

int ibm_nccl_unique_id(unsigned char out[128]) {
  if (!out) return IBM_ERR_ARG;
  ncclUniqueId id;
  if (ncclGetUniqueId(&id) != ncclSuccess) return IBM_ERR_NCCL;
  std::memcpy(out, id.internal, 128);
  return IBM_OK;
}

// Device-initiated halo across ranks (f3): every rank publishes a CUDA-IPC handle
// of the allocation holding its phi buffers (the caller's workspace) with their
// offsets and owned rows (NCCL all-gather); each rank maps its two neighbours'
// allocations.  All ranks then agree (all-reduce min) on whether every mapping
// succeeded: the peer-store passes and the NCCL-exchange passes issue different
// collectives, so either all ranks use them or none does.  Failure to map is not
// an error (the NCCL halo path stays in use); a failed collective is.
typedef CUresult (*PFN_memGetAddressRange)(CUdeviceptr *, size_t *, CUdeviceptr);
static int open_peer_halo(Ctx &c) {
  struct PeerInfo {
    cudaIpcMemHandle_t h;
    long long off[2];
    int nj, ok;
  };
  PeerInfo mine;
  std::memset(&mine, 0, sizeof(mine));
  static PFN_memGetAddressRange range_fn = nullptr;
  if (!range_fn) {
    void *p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuMemGetAddressRange", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      range_fn = reinterpret_cast<PFN_memGetAddressRange>(p);
  }
  const Slab &s0 = c.sl[0];
  CUdeviceptr base = 0;
  size_t size = 0;
  if (range_fn && range_fn(&base, &size, (CUdeviceptr)s0.phi[0]) == CUDA_SUCCESS &&
      cudaIpcGetMemHandle(&mine.h, (void *)base) == cudaSuccess) {
    mine.off[0] = (long long)((uintptr_t)s0.phi[0] - (uintptr_t)base);
    mine.off[1] = (long long)((uintptr_t)s0.phi[1] - (uintptr_t)base);
    mine.nj = s0.gp.nj;
    mine.ok = 1;
  }
  cudaGetLastError();  // (a failed IPC query is not sticky, but clear it)
  const size_t n = (size_t)c.nranks;
  char *d = nullptr;
  CK(cudaMalloc(&d, (n + 1) * sizeof(PeerInfo)));
  std::vector<PeerInfo> all(n);
  CK(cudaMemcpyAsync(d + n * sizeof(PeerInfo), &mine, sizeof(PeerInfo), cudaMemcpyHostToDevice, c.stream));
  NK(ncclAllGather(d + n * sizeof(PeerInfo), d, sizeof(PeerInfo), ncclChar, (ncclComm_t)c.nccl, c.stream));
  CK(cudaMemcpyAsync(all.data(), d, n * sizeof(PeerInfo), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  const int r = s0.rank;
  int ok = 1;
  for (int side = 0; side < 2 && ok; ++side) {
    const int nb = side == 0 ? r - 1 : r + 1;
    if (nb < 0 || nb >= c.nranks) continue;
    void *p = nullptr;
    if (!all[nb].ok || cudaIpcOpenMemHandle(&p, all[nb].h, cudaIpcMemLazyEnablePeerAccess) != cudaSuccess) {
      cudaGetLastError();
      ok = 0;
      break;
    }
    c.peer_map[side] = p;
    c.peer_phi[side][0] = (double *)((char *)p + all[nb].off[0]);
    c.peer_phi[side][1] = (double *)((char *)p + all[nb].off[1]);
    c.peer_nj[side] = all[nb].nj;
  }
  int *dok = reinterpret_cast<int *>(d);
  CK(cudaMemcpyAsync(dok, &ok, sizeof(int), cudaMemcpyHostToDevice, c.stream));
  NK(ncclAllReduce(dok, dok, 1, ncclInt32, ncclMin, (ncclComm_t)c.nccl, c.stream));
  CK(cudaMemcpyAsync(&ok, dok, sizeof(int), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  cudaFree(d);
  c.peer_halo = ok == 1;
  if (!c.peer_halo)
    for (int side = 0; side < 2; ++side) {
      if (c.peer_map[side]) cudaIpcCloseMemHandle(c.peer_map[side]);
      c.peer_map[side] = nullptr;
      c.peer_phi[side][0] = c.peer_phi[side][1] = nullptr;
    }
  return IBM_OK;
}

int ibm_init(const ibm_config *cfg, void *d_workspace, size_t bytes, void *cuda_stream, ibm_ctx **out) {
  if (!out) return IBM_ERR_ARG;
  *out = nullptr;
  std::string why;
  int st = check_config(cfg, why);
  if (st) {
    fprintf(stderr, "ibm_init: %s\n", why.c_str());
    return st;
  }
  ibm_ctx *cp = new (std::nothrow) ibm_ctx();
  if (!cp) return IBM_ERR_ARG;
  Ctx &c = *cp;
  c.cfg = *cfg;
  c.cfg.xn = c.cfg.yn = nullptr;
  c.cfg.nccl_id = nullptr;
  if (c.cfg.check_every < 1) c.cfg.check_every = 1;
  c.nx = cfg->nx;
  c.ny = cfg->ny;
  c.nranks = cfg->nranks;
  c.device = cfg->device;
  c.loopback = cfg->loopback;
  c.stream = (cudaStream_t)cuda_stream;
  c.nccl = nullptr;
  c.hint_uv = 16;
  c.hint_p = 64;
  // Poisson iterations fused per pass.  A decomposed grid exchanges 2m rows per
  // fused pass, so every slab must own that many; decided from cfg alone so that
  // all ranks agree (their collectives must match).
  // Automatic choice (sor_fuse = 0): m = 3 where the grid gives the fused pass
  // enough work items, else the one-iteration pass (wf_viable).
  c.wf_m = cfg->sor_fuse == 0 ? 3 : cfg->sor_fuse;
  // (the device first: wf_viable sizes the work-item target by its SM count)
  if (cudaSetDevice(c.device) != cudaSuccess) {
    fprintf(stderr, "ibm_init: cudaSetDevice failed\n");
    delete cp;
    return IBM_ERR_CUDA;
  }
  for (int r = 0; r < cfg->nranks; ++r) {
    int j0 = 0, j1 = cfg->ny;
    if (cfg->nranks > 1) slab_rows(cfg->ny, cfg->nranks, r, &j0, &j1);
    if (2 * c.wf_m > j1 - j0) c.wf_m = 1;
    if (cfg->sor_fuse == 0 && c.wf_m >= 2 && !wf_viable(cfg->nx, j1 - j0, c.wf_m)) c.wf_m = 1;
  }
  if (c.loopback)
    for (int r = 0; r < cfg->nranks; ++r) c.sl.push_back(make_slab(*cfg, r));
  else
    c.sl.push_back(make_slab(*cfg, cfg->rank));
  // every resource created below is released on any later failure
  for (auto &e : c.ev) e = nullptr;
  for (auto &e : c.tev) e = nullptr;
  c.h_ctl = nullptr;
  c.h_red = nullptr;
  c.h_nan = nullptr;
  c.comm = nullptr;
  c.ev_edge = c.ev_halo = nullptr;
  c.nccl_halo = nullptr;
  c.peer_halo = false;
  for (int q = 0; q < 2; ++q) {
    c.peer_phi[q][0] = c.peer_phi[q][1] = nullptr;
    c.peer_nj[q] = 0;
    c.peer_map[q] = nullptr;
  }
  auto fail = [&](int code) {
    fprintf(stderr, "ibm_init: %s\n", c.err.c_str());
    for (auto &e : c.ev)
      if (e) cudaEventDestroy(e);
    for (auto &e : c.tev)
      if (e) cudaEventDestroy(e);
    if (c.ev_edge) cudaEventDestroy(c.ev_edge);
    if (c.ev_halo) cudaEventDestroy(c.ev_halo);
    if (c.comm) cudaStreamDestroy(c.comm);
    if (c.nccl_halo) ncclCommDestroy((ncclComm_t)c.nccl_halo);
    if (c.nccl) ncclCommDestroy((ncclComm_t)c.nccl);
    if (c.h_ctl) cudaFreeHost(c.h_ctl);
    if (c.h_red) cudaFreeHost(c.h_red);
    if (c.h_nan) cudaFreeHost(c.h_nan);
    for (auto &p : c.peer_map)
      if (p) cudaIpcCloseMemHandle(p);
    delete cp;
    return code;
  };
  const size_t need = carve(c, nullptr);
  if (!d_workspace || bytes < need || ((uintptr_t)d_workspace & 255)) {
    c.err = "workspace NULL, misaligned or too small (need " + std::to_string(need) + " B)";
    return fail(IBM_ERR_ARG);
  }
  carve(c, (char *)d_workspace);
  if (!make_coef_maps(c)) return fail(IBM_ERR_CUDA);
  for (Slab &s : c.sl)
    if (!make_maps(s, c.wf_m)) {
      c.err = "cuTensorMapEncodeTiled unavailable or failed";
      return fail(IBM_ERR_CUDA);
    }
  if (cudaHostAlloc((void **)&c.h_ctl, 2 * sizeof(SorCtl), cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc((void **)&c.h_red, 4 * sizeof(double) * c.sl.size(), cudaHostAllocDefault) != cudaSuccess ||
      cudaHostAlloc((void **)&c.h_nan, sizeof(int), cudaHostAllocDefault) != cudaSuccess) {
    c.err = "cudaHostAlloc failed";
    return fail(IBM_ERR_CUDA);
  }
  for (auto &e : c.ev)
    if (cudaEventCreate(&e) != cudaSuccess) { c.err = "cudaEventCreate failed"; return fail(IBM_ERR_CUDA); }
  for (auto &e : c.tev)
    if (cudaEventCreate(&e) != cudaSuccess) { c.err = "cudaEventCreate failed"; return fail(IBM_ERR_CUDA); }
  if (c.sl.size() > 1 || c.nranks > 1) {  // decomposed: the overlapped halo exchange of the fused pass
    if (cudaStreamCreateWithFlags(&c.comm, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.ev_edge, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&c.ev_halo, cudaEventDisableTiming) != cudaSuccess) {
      c.err = "comm stream / events";
      return fail(IBM_ERR_CUDA);
    }
  }
  c.wf_L = 0;
  // mid-size single-slab grids without the fused pass: resident temporally blocked
  // Poisson solve when its tiles fit the co-resident grid (IBM_SOR_TB=0 disables,
  // IBM_SOR_TB=m picks the iterations per grid barrier, default 4)
  c.tb_m = 0;
  {
    const char *e = std::getenv("IBM_SOR_TB");
    const int m = e ? std::atoi(e) : 4;
    if (m >= 2 && c.wf_m == 1 && c.sl.size() == 1 && c.nranks == 1) {
      int sms = 0;
      cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, c.device);
      std::memset(&c.tb, 0, sizeof(c.tb));
      const Slab &s = c.sl[0];
      c.tb.g = s.gp;
      c.tb.cE = c.m.cEp; c.tb.cW = c.m.cWp; c.tb.cD = c.m.cDp; c.tb.cN = c.m.cNp; c.tb.cS = c.m.cSp;
      c.tb.ui0 = 0; c.tb.ui1 = c.nx; c.tb.uj0 = 0; c.tb.uj1 = c.ny;
      // (deeper blocking needs wider halos: fall back to fewer iterations per barrier
      // when the tiles of m do not fit the co-resident grid)
      for (int mm = std::min(m, 4); mm >= 2 && c.tb_m == 0 && sms > 0; --mm)
        if (tb_plan(c.tb, c.nx, s.gp.nj, mm, sms)) c.tb_m = mm;
    }
  }
  HostMetric h = host_metric(*cfg);
  c.h_cNp = h.cNp;
  c.h_cSp = h.cSp;
  c.h_xn = nullptr;
  c.h_yn = nullptr;
  auto up = [&](double *d, const std::vector<double> &v) {
    return cudaMemcpyAsync(d, v.data(), v.size() * sizeof(double), cudaMemcpyHostToDevice, c.stream);
  };
  cudaError_t e = cudaMemsetAsync(d_workspace, 0, need, c.stream);
  const Metric &m = c.m;
  const std::pair<double *, const std::vector<double> *> ups[] = {
      {m.xn, &h.xn}, {m.yn, &h.yn}, {m.dx, &h.dx}, {m.dy, &h.dy}, {m.xc, &h.xc}, {m.yc, &h.yc},
      {m.hxc, &h.hxc}, {m.hyc, &h.hyc}, {m.cEu, &h.cEu}, {m.cWu, &h.cWu}, {m.cDu, &h.cDu},
      {m.cNu, &h.cNu}, {m.cSu, &h.cSu}, {m.cEv, &h.cEv}, {m.cWv, &h.cWv}, {m.cDv, &h.cDv},
      {m.cNv, &h.cNv}, {m.cSv, &h.cSv}, {m.cEp, &h.cEp}, {m.cWp, &h.cWp}, {m.cDp, &h.cDp},
      {m.cNp, &h.cNp}, {m.cSp, &h.cSp}};
  for (auto &pr : ups)
    if (e == cudaSuccess) e = up(pr.first, *pr.second);
  if (e == cudaSuccess)
    for (Slab &s : c.sl) launch_fill(s.u, s.gu, 1.0, c.stream);  // impulsive start (R11)
  if (e == cudaSuccess) e = cudaStreamSynchronize(c.stream);
  if (e != cudaSuccess) {
    c.err = std::string("init upload: ") + cudaGetErrorString(e);
    return fail(IBM_ERR_CUDA);
  }
  if (c.nranks > 1 && !c.loopback) {
    ncclUniqueId id;
    std::memcpy(id.internal, cfg->nccl_id, 128);
    ncclComm_t comm;
    ncclResult_t nr = ncclCommInitRank(&comm, c.nranks, id, cfg->rank);
    if (nr != ncclSuccess) {
      c.err = std::string("ncclCommInitRank: ") + ncclGetErrorString(nr);
      return fail(IBM_ERR_NCCL);
    }
    c.nccl = comm;
    ncclComm_t halo_comm;
    nr = ncclCommSplit(comm, 0, cfg->rank, &halo_comm, nullptr);
    if (nr != ncclSuccess) {
      c.err = std::string("ncclCommSplit: ") + ncclGetErrorString(nr);
      return fail(IBM_ERR_NCCL);
    }
    c.nccl_halo = halo_comm;
  }
  {
    const char *e = std::getenv("IBM_PEER_HALO");
    const bool want = !(e && std::atoi(e) == 0);
    if (c.loopback) c.peer_halo = want && c.sl.size() > 1;
    else if (c.nranks > 1 && want && c.wf_m >= 2)
      if (int st = open_peer_halo(c)) return fail(st);
  }
  c.body = Body{0, 0, 0, 0, 0, 0, 0};
  c.phi_cur = 0;
  c.step = 0;
  c.have_hist = 0;
  c.Mx = c.My = 0.0;
  c.last_t = c.last_cd = c.last_cl = 0.0;
  // host copies of the family coordinates for the body boxes
  c.h_xn = new double[c.nx + 1];
  c.h_yn = new double[c.ny + 1];
  std::memcpy(c.h_xn, cfg->xn, sizeof(double) * (c.nx + 1));
  std::memcpy(c.h_yn, cfg->yn, sizeof(double) * (c.ny + 1));
  *out = cp;
  return IBM_OK;
}

static int set_body_impl(ibm_ctx *ctx, const Body &B) {
  Ctx &c = *ctx;
  CK(cudaSetDevice(c.device));
  const int nx = c.nx, ny = c.ny;
  const double *xn = c.h_xn, *yn = c.h_yn;
  // zero tags, flags and forcing fields of the previous body
  for (Slab &s : c.sl) {
    CK(cudaMemsetAsync(s.tu, 0, s.gu.elems(), c.stream));
    CK(cudaMemsetAsync(s.tv, 0, s.gv.elems(), c.stream));
    CK(cudaMemsetAsync(s.tp, 0, s.gp.elems(), c.stream));
    CK(cudaMemsetAsync(s.pf, 0, s.gp.elems(), c.stream));
    CK(cudaMemsetAsync(s.fu, 0, s.gu.elems() * sizeof(double), c.stream));
    CK(cudaMemsetAsync(s.fv, 0, s.gv.elems() * sizeof(double), c.stream));
    s.bu = s.bv = s.bpb = BBox{0, 0, 0, 0};
  }
  c.body = B;
  if (B.has) {
    std::vector<double> vxn(xn, xn + nx + 1), vyn(yn, yn + ny + 1), vxc(nx), vyc(ny);
    for (int i = 0; i < nx; ++i) vxc[i] = 0.5 * (xn[i] + xn[i + 1]);
    for (int j = 0; j < ny; ++j) vyc[j] = 0.5 * (yn[j] + yn[j + 1]);
    const double xlo = B.x0 - B.a, xhi = B.x0 + B.a;
    const double ylo = B.y0 - B.hbar - B.b, yhi = B.y0 + B.hbar + B.b;
    for (Slab &s : c.sl) {
      s.bu = box_for(vxn, vyc, xlo, xhi, ylo, yhi, s.gu, 3);
      s.bv = box_for(vxc, vyn, xlo, xhi, ylo, yhi, s.gv, 3);
      s.bpb = box_for(vxc, vyc, xlo, xhi, ylo, yhi, s.gp, 3);
    }
  }
  return refresh_time(c);
}

int ibm_set_body(ibm_ctx *ctx, double a, double b, double x0, double y0, double h_bar, double k) {
  if (!ctx) return IBM_ERR_ARG;
  Ctx &c = *ctx;
  if (!(a > 0) || !(b > 0) || !(k > 0) || !(h_bar >= 0)) {
    c.err = "body: a, b, k must be > 0 and h_bar >= 0";
    return IBM_ERR_CONFIG;
  }
  const double *xn = c.h_xn, *yn = c.h_yn;
  if (!(x0 - a > xn[3] && x0 + a < xn[c.nx - 3] && y0 - h_bar - b > yn[3] && y0 + h_bar + b < yn[c.ny - 3])) {
    c.err = "body envelope must lie inside the domain by >= 3 cells";
    return IBM_ERR_CONFIG;
  }
  return set_body_impl(ctx, Body{1, a, b, x0, y0, h_bar, k});
}

int ibm_clear_body(ibm_ctx *ctx) {
  if (!ctx) return IBM_ERR_ARG;
  return set_body_impl(ctx, Body{0, 0, 0, 0, 0, 0, 0});
}

// per-field device pointer / family geometry / element size
static bool field_of(Slab &s, int bit, int phi_cur, void **ptr, const Geo **g, size_t *esz) {
  *esz = sizeof(double);
  switch (bit) {
    case 0: *ptr = s.u; *g = &s.gu; return true;
    case 1: *ptr = s.v; *g = &s.gv; return true;
    case 2: *ptr = s.p; *g = &s.gp; return true;
    case 3: *ptr = s.phi[phi_cur]; *g = &s.gp; return true;
    case 4: *ptr = s.fu; *g = &s.gu; return true;
    case 5: *ptr = s.fv; *g = &s.gv; return true;
    case 6: *ptr = s.q; *g = &s.gp; return true;
    case 7: *ptr = s.tu; *g = &s.gu; *esz = 1; return true;
    case 8: *ptr = s.tv; *g = &s.gv; *esz = 1; return true;
    case 9: *ptr = s.tp; *g = &s.gp; *esz = 1; return true;
    case 10: *ptr = s.cup; *g = &s.gu; return true;
    case 11: *ptr = s.cvp; *g = &s.gv; return true;
  }
  return false;
}

static int copy_fields(Ctx &c, unsigned mask, void *const *dst, const void *const *src, int where, bool get) {
  const int base_row = c.loopback ? 0 : c.sl[0].pj0;
  for (int bit = 0; bit < IBM_NFIELDS; ++bit) {
    if (!(mask & (1u << bit))) continue;
    void *user = get ? dst[bit] : const_cast<void *>(src[bit]);
    if (!user) { c.err = "NULL buffer for field bit " + std::to_string(bit); return IBM_ERR_ARG; }
    for (Slab &s : c.sl) {
      void *dptr;
      const Geo *g;
      size_t esz;
      field_of(s, bit, c.phi_cur, &dptr, &g, &esz);
      char *dev = (char *)dptr + (size_t)g->off(0, 0) * esz;
      char *hst = (char *)user + (size_t)(g->gj0 - base_row) * g->ni * esz;
      const size_t wb = (size_t)g->ni * esz, pb = (size_t)g->pitch * esz;
      cudaMemcpyKind kind = where == IBM_HOST ? (get ? cudaMemcpyDeviceToHost : cudaMemcpyHostToDevice)
                                              : cudaMemcpyDeviceToDevice;
      if (get)
        CK(cudaMemcpy2DAsync(hst, wb, dev, pb, wb, g->nj, kind, c.stream));
      else
        CK(cudaMemcpy2DAsync(dev, pb, hst, wb, wb, g->nj, kind, c.stream));
    }
  }
  CK(cudaStreamSynchronize(c.stream));
  return IBM_OK;
}

int ibm_set_fields(ibm_ctx *ctx, unsigned mask, const void *const *src, int where) {
  if (!ctx) return IBM_ERR_ARG;
  Ctx &c = *ctx;
  const unsigned ok = IBM_U | IBM_V | IBM_P | IBM_PHI | IBM_CU_PREV | IBM_CV_PREV;
  if (!src || (mask & ~ok)) { c.err = "set_fields: bad mask or NULL src"; return IBM_ERR_ARG; }
  CK(cudaSetDevice(c.device));
  return copy_fields(c, mask, nullptr, src, where, false);
}

int ibm_set_step(ibm_ctx *ctx, int step, int have_history) {
  if (!ctx) return IBM_ERR_ARG;
  Ctx &c = *ctx;
  if (step < 0) { c.err = "step < 0"; return IBM_ERR_ARG; }
  CK(cudaSetDevice(c.device));
  c.step = step;
  c.have_hist = have_history ? 1 : 0;
  return refresh_time(c);
}

int ibm_step(ibm_ctx *ctx, int nsteps, ibm_step_stats *stats) {
  if (!ctx) return IBM_ERR_STATE;
  Ctx &c = *ctx;
  if (nsteps < 0) return IBM_ERR_ARG;
  CK(cudaSetDevice(c.device));
  int worst = IBM_OK;
  for (int n = 0; n < nsteps; ++n) {
    ibm_step_stats local;
    std::memset(&local, 0, sizeof(local));
    int st = step_once(c, &local);
    local.status = st;
    if (stats) stats[n] = local;
    if (st == IBM_ERR_DIVERGED || st > IBM_ERR_DIVERGED) return st;
    if (st > worst) worst = st;
  }
  return worst;
}

int ibm_get_fields(ibm_ctx *ctx, unsigned mask, void *const *dst, int where, int *j0, int *j1) {
  if (!ctx) return IBM_ERR_ARG;
  Ctx &c = *ctx;
  if (!dst || (mask >> IBM_NFIELDS)) { c.err = "get_fields: bad mask or NULL dst"; return IBM_ERR_ARG; }
  CK(cudaSetDevice(c.device));
  if (j0) *j0 = c.loopback ? 0 : c.sl[0].pj0;
  if (j1) *j1 = c.loopback ? c.ny : c.sl[0].pj1;
  return copy_fields(c, mask, dst, nullptr, where, true);
}

int ibm_forces(ibm_ctx *ctx, double out[3]) {
  if (!ctx || !out) return IBM_ERR_ARG;
  out[0] = ctx->last_t;
  out[1] = ctx->last_cd;
  out[2] = ctx->last_cl;
  return IBM_OK;
}

int ibm_poisson_iterate(ibm_ctx *ctx, int iters, double *rho_out) {
  if (!ctx) return IBM_ERR_STATE;
  Ctx &c = *ctx;
  if (iters < 1 || (size_t)iters + 2 > rho_len(c.cfg)) { c.err = "iters outside [1, max(maxit)]"; return IBM_ERR_ARG; }
  CK(cudaSetDevice(c.device));
  int k = 0, sst = 0;
  double rho = 0.0;
  int pbuf = c.phi_cur;
  int r = sor_solve(c, false, c.phi_cur, &k, &rho, &sst, iters, &pbuf);
  if (r) return r;
  c.phi_cur = pbuf;
  if (rho_out) *rho_out = rho;
  return sst == 3 ? IBM_ERR_DIVERGED : IBM_OK;
}

int ibm_query(const ibm_ctx *ctx, int key, int *out) {
  if (!ctx || !out) return IBM_ERR_ARG;
  switch (key) {
    case IBM_QUERY_WF_M: *out = ctx->wf_m; return IBM_OK;
    case IBM_QUERY_WF_L: *out = ctx->wf_L; return IBM_OK;
    case IBM_QUERY_SLABS: *out = (int)ctx->sl.size(); return IBM_OK;
    case IBM_QUERY_TB_M: *out = ctx->tb_m; return IBM_OK;
    case IBM_QUERY_PEER_HALO: *out = ctx->peer_halo ? 1 : 0; return IBM_OK;
  }
  return IBM_ERR_ARG;
}

const char *ibm_last_error(const ibm_ctx *ctx) {
  if (!ctx) return kNoCtx;
  return ctx->err.c_str();
}

int ibm_destroy(ibm_ctx *ctx) {
  if (!ctx) return IBM_ERR_ARG;
  Ctx &c = *ctx;
  cudaSetDevice(c.device);
  cudaStreamSynchronize(c.stream);
  if (c.comm) cudaStreamSynchronize(c.comm);
  if (c.nccl_halo) ncclCommDestroy((ncclComm_t)c.nccl_halo);
  if (c.nccl) ncclCommDestroy((ncclComm_t)c.nccl);
  if (c.ev_edge) cudaEventDestroy(c.ev_edge);
  if (c.ev_halo) cudaEventDestroy(c.ev_halo);
  if (c.comm) cudaStreamDestroy(c.comm);
  for (auto &e : c.ev) cudaEventDestroy(e);
  for (auto &e : c.tev) cudaEventDestroy(e);
  cudaFreeHost(c.h_ctl);
  cudaFreeHost(c.h_red);
  cudaFreeHost(c.h_nan);
  for (auto &kv : c.wf_segs) cudaFree(kv.second.second);
  for (auto &p : c.peer_map)
    if (p) cudaIpcCloseMemHandle(p);
  delete[] c.h_xn;
  delete[] c.h_yn;
  delete ctx;
  return IBM_OK;
}

}  // extern "C"
