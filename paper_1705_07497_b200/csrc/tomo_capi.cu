// tomo_capi.cu — host runtime (C++) and C ABI of libtomo_b200.so.
//
// Mirrors the reference's operator/solver API (proj/include/tomo/*.hpp): geometry + plan
// construction (fourier_slice.cpp:10-48, nufft.cpp:26-101) in fp64 on the host, the W / W^T
// sparse tables in device HBM, and the apply / CG / split-Bregman / Tikhonov drivers
// (normal_ops.cpp:321-340, solver.cpp:56-337) as sequences of sm_100a kernels, captured into
// CUDA graphs for the iterative loops. No compute runs on the host: every hot-path call
// requires the CUDA kernels and fails with TOMO_ERR_CUDA if they cannot run.
//
// An op has one precision (fp32: complex64 data, or fp64: complex128 data) fixed at
// creation; all drivers are templates over the real type R and dispatched at the ABI.
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <atomic>
#include <condition_variable>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <map>
#include <mutex>
#include <tuple>
#include <memory>
#include <random>
#include <stdexcept>
#include <string>
#include <vector>

#include "../../include/tomo_b200.h"
#include "kernels.h"
#include "tspm.h"

namespace tomo_b200 {

struct ConfigError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct NumericalError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct CudaError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
struct IoError : std::runtime_error {
  using std::runtime_error::runtime_error;
};
using TspmIO = Tspm<IoError, ConfigError>;

thread_local std::string g_err;
std::atomic<int64_t> g_launches{0};
thread_local int64_t* g_capture_count = nullptr;

void check_launch(cudaError_t e) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw CudaError(std::string("kernel launch failed: ") + cudaGetErrorString(e));
  }
}

void note_launch() {
  if (g_capture_count)
    ++*g_capture_count;
  else
    g_launches.fetch_add(1, std::memory_order_relaxed);
  const cudaError_t e = cudaPeekAtLastError();
  if (e != cudaSuccess) {
    cudaGetLastError();
    throw CudaError(std::string("kernel launch failed: ") + cudaGetErrorString(e));
  }
}

#define CK(x)                                                                                  \
  do {                                                                                         \
    const cudaError_t e_ = (x);                                                                \
    if (e_ != cudaSuccess) throw CudaError(std::string(#x) + ": " + cudaGetErrorString(e_)); \
  } while (0)

// Raw device allocation, viewed as any element type.
struct Raw {
  void* p = nullptr;
  size_t bytes = 0;
  Raw() = default;
  Raw(const Raw&) = delete;
  Raw& operator=(const Raw&) = delete;
  ~Raw() { release(); }
  void release() {
    if (p) cudaFree(p);
    p = nullptr;
    bytes = 0;
  }
  void ensure(size_t nbytes) {
    if (nbytes <= bytes) return;
    release();
    CK(cudaMalloc(&p, std::max<size_t>(nbytes, 16)));
    bytes = nbytes;
  }
  template <typename T>
  T* as() const {
    return static_cast<T*>(p);
  }
  template <typename T>
  void upload(const std::vector<T>& v) {
    ensure(v.size() * sizeof(T));
    CK(cudaMemcpy(p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice));
  }
};

struct DeviceGuard {
  int prev = -1;
  explicit DeviceGuard(int dev) {
    CK(cudaGetDevice(&prev));
    if (prev != dev) CK(cudaSetDevice(dev));
  }
  ~DeviceGuard() {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != prev && prev >= 0) cudaSetDevice(prev);
  }
};

bool is_device_ptr(const void* p) {
  if (!p) return false;
  cudaPointerAttributes a{};
  if (cudaPointerGetAttributes(&a, p) != cudaSuccess) {
    cudaGetLastError();
    return false;
  }
  return a.type == cudaMemoryTypeDevice || a.type == cudaMemoryTypeManaged;
}

// ------------------------------------------------------------------------------------------
// Geometry (fp64 host): make_angle_set / slice_points (fourier_slice.cpp:10-41) with n_b
// radial samples, FrequencyPointSet::make (nufft.cpp:43-54), plan_spreading (:71-101) and
// SpreadingPlan::weights (:56-69) over the window [lo, hi].
// ------------------------------------------------------------------------------------------
struct Geom {
  int n = 0, A = 0, nb = 0, R = 2, lo = 0, hi = 0, m = 0, w = 0;
  double tau = 0.0;
  std::vector<double> angles;
  int a0 = 0, a1 = 0;  // local angle block
  int64_t P = 0;       // local samples
};

Geom make_geom(const tomo_geom_desc* d, const tomo_op_desc* od) {
  if (!d) throw ConfigError("geometry: null descriptor");
  Geom g;
  g.n = d->n;
  g.A = d->n_angles;
  g.nb = d->n_b > 0 ? d->n_b : d->n;
  g.R = d->oversample > 0 ? d->oversample : 2;
  g.lo = d->win_lo;
  g.hi = d->win_hi;
  g.tau = d->tau;
  if (g.n < 4) throw ConfigError("make_params: n must be >= 4");
  if (g.n % 2 != 0) throw ConfigError("slice_points: n must be even");
  if (g.A < 1) throw ConfigError("geometry: need at least one angle");
  if (g.nb < 2) throw ConfigError("geometry: n_b must be >= 2");
  if (g.R < 2) throw ConfigError("geometry: oversampling must be >= 2");
  if (!(g.lo <= 0 && g.hi >= 0)) throw ConfigError("geometry: window must contain 0");
  if (!(g.tau > 0.0)) throw ConfigError("make_params: tau must be positive");
  g.m = g.R * g.n;
  g.w = g.hi - g.lo + 1;
  if (g.w > 64) throw ConfigError("spreading window too wide (max 64 taps per axis)");
  if (g.w > g.R * g.n) throw ConfigError("spreading window wider than the oversampled grid");
  if (g.m < 32 || g.m > 8192 || (g.m & (g.m - 1)) != 0)
    throw ConfigError("grid side m = R*n must be a power of two in [32, 8192]");
  g.angles.resize(g.A);
  for (int a = 0; a < g.A; ++a) g.angles[a] = d->angles ? d->angles[a] : a * M_PI / g.A;
  g.a0 = 0;
  g.a1 = g.A;
  if (od && (od->angle_begin != 0 || od->angle_end != 0)) {
    if (od->angle_begin < 0 || od->angle_end > g.A || od->angle_begin >= od->angle_end)
      throw ConfigError("op: bad angle block");
    g.a0 = od->angle_begin;
    g.a1 = od->angle_end;
  }
  g.P = static_cast<int64_t>(g.a1 - g.a0) * g.nb;
  if (static_cast<int64_t>(g.m) * g.m * 8 > (int64_t(1) << 40)) throw ConfigError("grid too large");
  return g;
}

struct Plan {
  std::vector<int> mjx, mjy;
  std::vector<double> wx, wy;  // P x w
};

Plan make_plan(const Geom& g) {
  Plan pl;
  pl.mjx.resize(g.P);
  pl.mjy.resize(g.P);
  pl.wx.resize(g.P * g.w);
  pl.wy.resize(g.P * g.w);
  constexpr double two_pi = 2.0 * M_PI;
  const double big_m = g.m / 2.0, h = M_PI / big_m, tau = g.tau;
  std::vector<double> e3(g.w);
  for (int l = g.lo; l <= g.hi; ++l) e3[l - g.lo] = std::exp(-(M_PI * l / big_m) * (M_PI * l / big_m) / (4.0 * tau));
  auto reduce = [](double v) {
    double r = std::fmod(v, two_pi);
    if (r < 0.0) r += two_pi;
    if (r >= two_pi) r = 0.0;
    return r;
  };
  const int reach = std::max(g.hi, -g.lo);
  int64_t j = 0;
  for (int a = g.a0; a < g.a1; ++a) {
    const double c = std::cos(g.angles[a]), s = std::sin(g.angles[a]);
    for (int t = 0; t < g.nb; ++t, ++j) {
      const double k_r = (2.0 * M_PI / g.nb) * (t - g.nb / 2);
      const double xy[2] = {reduce(k_r * c), reduce(k_r * s)};
      for (int dd = 0; dd < 2; ++dd) {
        int mj = static_cast<int>(std::floor(xy[dd] / h));
        if (mj >= g.m) mj = g.m - 1;
        const double xi = xy[dd] - h * mj;
        const double f1 = std::exp(-xi * xi / (4.0 * tau));
        const double f2 = std::exp(xi * M_PI / (big_m * 2.0 * tau));
        const double f2inv = 1.0 / f2;
        double* w = (dd == 0 ? pl.wx.data() : pl.wy.data()) + j * g.w;
        w[-g.lo] = f1;
        double p = f1, q = f1;
        for (int l = 1; l <= reach; ++l) {
          p *= f2;
          q *= f2inv;
          if (l <= g.hi) w[l - g.lo] = p * e3[l - g.lo];
          if (-l >= g.lo) w[-l - g.lo] = q * e3[-l - g.lo];
        }
        (dd == 0 ? pl.mjx : pl.mjy)[j] = mj;
      }
    }
  }
  return pl;
}

inline int wrapi(int idx, int m) { return idx < 0 ? idx + m : (idx >= m ? idx - m : idx); }

constexpr int kMaxLoggedIters = 8192;

// Device scratch of an op, sized for `cap` slices (element type = op precision).
struct Scratch {
  int cap = 0;
  Raw H, g, s, K, Gt, Gth, part_wt, part_gram;  // complex (Gth: the folded half grid, own buffer)
  Raw heavy_cnt, heavy_cnt_gram;
  Raw cin, cout, fin, fout;       // staging for host pointers / temporaries
  Raw r, p0, p1, ap, x, rhs, fid, mu0, mu1, bx0, bx1, by0, by1, nred, zero, u2;  // real vectors
  Raw upd_log, rel_log, sc, part;
  Raw fk, fint;  // split-Bregman data feedback: running data and the slice data, internal order
};

// Device tables of one task-SpMV operator (the fused backend's Gram; see TaskSpmv).
struct TaskSet {
  Raw ent, tasks, perm, heavy, slot_heavy;
  int n_tasks = 0, n_heavy = 0, n_slots = 0;
  int64_t slots = 0, nnz = 0, bytes = 0, touched = 0;
};

struct GraphEntry {
  cudaGraphExec_t exec = nullptr;
  int64_t nodes = 0;
};

// Mutable per-call state of an op: device scratch, execution lanes, host-copy pipeline and the
// CUDA graphs captured over that scratch. The op itself (geometry, W / W^T / Gram / stencil
// tables) is immutable after creation and shared; every API call leases one workspace for its
// stream (Lease below), so concurrent calls on distinct streams use distinct workspaces
// (built operators are shareable, concurrent solves on separate state are
// safe).
struct Workspace {
  static constexpr int kMaxLanes = 4;
  Scratch sc;
  // extra execution lanes for batches of independent slices (apply paths): each has its own
  // grids, W^T partial/ticket buffers and stream, so sub-batches run concurrently
  Scratch lanes[kMaxLanes - 1];  // lanes 1..kMaxLanes-1 (lane 0 = sc)
  int cur_lane = 0;              // dev() hands out lane cur_lane's buffers
  cudaStream_t lane_st[kMaxLanes - 1] = {};
  cudaEvent_t lane_fork = nullptr, lane_join[kMaxLanes - 1] = {};
  // host-buffer pipeline (host_pipeline): copy streams, events, double-buffered staging
  cudaStream_t pipe_in = nullptr, pipe_out = nullptr;
  cudaEvent_t ev_in[2] = {nullptr, nullptr}, ev_comp[2] = {nullptr, nullptr}, ev_out[2] = {nullptr, nullptr};
  Raw pin_buf[2], pout_buf[2];
  std::map<std::string, GraphEntry> graphs;
  // lease bookkeeping: the stream of the last call and an event recorded there when it returned
  cudaStream_t last_stream = nullptr;
  cudaEvent_t done = nullptr;
  bool busy = false;
  bool captured = false;  // used inside a caller's stream capture: reserved for that stream
  uint64_t last_use = 0;

  Workspace() = default;
  Workspace(const Workspace&) = delete;
  Workspace& operator=(const Workspace&) = delete;
  ~Workspace() {
    clear_graphs();
    for (int k = 0; k < 2; ++k)
      for (cudaEvent_t e : {ev_in[k], ev_comp[k], ev_out[k]})
        if (e) cudaEventDestroy(e);
    if (pipe_in) cudaStreamDestroy(pipe_in);
    if (pipe_out) cudaStreamDestroy(pipe_out);
    if (lane_fork) cudaEventDestroy(lane_fork);
    if (done) cudaEventDestroy(done);
    for (int k = 0; k < kMaxLanes - 1; ++k) {
      if (lane_join[k]) cudaEventDestroy(lane_join[k]);
      if (lane_st[k]) cudaStreamDestroy(lane_st[k]);
    }
  }
  void clear_graphs() {
    for (auto& kv : graphs)
      if (kv.second.exec) cudaGraphExecDestroy(kv.second.exec);
    graphs.clear();
  }
};

}  // namespace tomo_b200

using namespace tomo_b200;

struct tomo_op {
  Geom g;
  tomo_op_desc desc{};
  int device = 0;
  bool f64 = false;
  size_t rsz = 4;  // sizeof(R)
  int64_t nnz = 0, wt_rows = 0, wt_slots = 0;
  int Ppad = 0;
  int n_tasks = 0, n_heavy = 0, n_slots = 0;
  Raw apod, tw, twh, wbase, wxs, wys, wtent, wttasks, wtperm, wtheavy, wtslotheavy;
  Raw wperm;           // separable-W table position -> sample (grid-tile order)
  bool w_sorted = false;
  TaskSet gram;  // fused backend only
  TaskSet herm;  // W^T folded onto grid rows [0, m/2] (real-subspace type-1); n_tasks == 0: not built
  // Mirror pairs (opbuild.cu): for real images the normal operator needs W on one sample of every
  // mirror pair only (half W: hbase / hwx / hwy, Ph samples) and the folded W^T of the primaries
  // (sym); used by normal_core when both ends are real. n_tasks == 0: not built (no pairs).
  // sym_mode 1: mirror-image windows (lo = 1 - hi). sym_mode 2 ("overlap pairs", the reference's
  // [-m_sp, m_sp]): the partner's window is the mirror image shifted by one node, so W stays whole,
  // a small kernel forms the pair sums s_j + conj(s_partner) behind the samples (ppos: partner
  // positions) and the fold reads them inside the pairs' common window.
  TaskSet sym;
  Raw pairs, hbase, hwx, hwy, ppos;
  // overlap pairs, W by units (PairW; built for windows of at most 7 nodes): hbase / hwx / hwy hold
  // the unit tables ((w + 1) factors per axis), upos / uppos the output positions
  Raw upos, uppos;
  int64_t n_units = 0;
  int Upad = 0;
  template <typename R>
  PairW<R> pair_w() const {
    return PairW<R>{static_cast<int>(n_units), Upad, hbase.as<int>(), hwx.as<R>(), hwy.as<R>(), upos.as<int>(),
                    uppos.as<int>()};
  }
  int64_t Ph = 0, n_paired = 0;
  int Ppad_h = 0;
  int sym_mode = 0;
  const TspmFile* src = nullptr;  // during tomo_op_create_tspm: the loaded Gram / surrogate T
  // surrogate
  int rad = 0;
  StencilCoef coef{};
  double stencil64[81] = {0};
  // lazily computed, per-op caches (shared by every workspace; guarded by cache_mu)
  std::mutex cache_mu;
  std::map<std::pair<double, double>, double> sigma_cache;
  double leak = -1.0;
  // collective
  tomo_allreduce_fn ar_fn = nullptr;
  void* ar_user = nullptr;
  ncclComm_t comm = nullptr;
  // workspaces (Lease): at most kMaxWorkspaces, one per concurrently calling stream
  static constexpr int kMaxLanes = Workspace::kMaxLanes;
  static constexpr int kMaxWorkspaces = 8;
  std::mutex ws_mu;
  std::condition_variable ws_cv;
  std::vector<std::unique_ptr<Workspace>> pool;
  uint64_t ws_clock = 0;

  ~tomo_op() {
    pool.clear();
    if (comm) ncclCommDestroy(comm);
  }
  // the workspace leased by the calling thread (every scratch-touching entry point holds one)
  Workspace& W() const;
  void clear_graphs() { W().clear_graphs(); }
  void clear_all_graphs() {
    std::lock_guard<std::mutex> lk(ws_mu);
    for (auto& w : pool) w->clear_graphs();
  }

  bool sharded() const { return g.a0 != 0 || g.a1 != g.A; }
  // real-subspace (Hermitian half-grid) pipeline available: folded W^T built, pairs of image rows
  bool herm_ok() const { return herm.n_tasks > 0 && g.n % 2 == 0; }
  bool sym_ok() const { return herm_ok() && sym.n_tasks > 0 && sym_mode > 0; }
  // sample vector entries per slice (overlap pairs keep the pair sums behind the samples)
  size_t s_len() const { return static_cast<size_t>(g.P) * (sym_mode == 2 ? 2 : 1); }
  // the real-subspace normal operator through the mirror pairs: W on the half sample set (written
  // at its compact positions), the primaries' folded W^T reading those positions
  template <typename R>
  void use_sym(OpDev<R>& d) const {
    d.wth = TaskSpmv<R>{sym.ent.as<WtEnt<R>>(), sym.tasks.as<int4>(), sym.n_tasks, sym.perm.as<uint16_t>(),
                        sym.heavy.as<int4>(), sym.slot_heavy.as<int>(), d.wth.heavy_cnt, sym.n_heavy, sym.n_slots,
                        d.wth.part};
    if (sym_mode == 2) {
      d.s_stride = 2 * d.P;
      return;
    }
    d.w_base = hbase.as<int>();
    d.w_x = hwx.as<R>();
    d.w_y = hwy.as<R>();
    d.w_perm = nullptr;
    d.w_out_pos = 1;
    d.P = static_cast<int>(Ph);
    d.Ppad = Ppad_h;
    d.s_stride = d.P;
  }
  bool surrogate() const { return desc.backend == TOMO_BACKEND_SURROGATE; }
  bool fused() const { return desc.backend == TOMO_BACKEND_FUSED; }
  int64_t L() const { return static_cast<int64_t>(g.n) * g.n; }

  template <typename R>
  OpDev<R> dev(int B) {
    ensure_batch(B);
    Workspace& ws = W();
    if (ws.cur_lane) ensure_lane(ws.cur_lane, B);
    Scratch& sc = ws.cur_lane ? ws.lanes[ws.cur_lane - 1] : ws.sc;
    OpDev<R> d{};
    d.n = g.n;
    d.m = g.m;
    d.nb = g.nb;
    d.P = static_cast<int>(g.P);
    d.s_stride = d.P;
    d.Ppad = Ppad;
    d.G32 = static_cast<int>(static_cast<int64_t>(g.m) * g.m / 32);
    d.apod = apod.as<R>();
    d.tw = tw.as<cplx<R>>();
    d.tw_half = twh.as<cplx<R>>();
    d.w_base = wbase.as<int>();
    d.w_x = wxs.as<R>();
    d.w_y = wys.as<R>();
    d.w_perm = w_sorted ? wperm.as<int>() : nullptr;
    d.w_out_pos = w_sorted ? 1 : 0;
    d.w = g.w;
    d.wt_ent = wtent.as<WtEnt<R>>();
    d.wt_tasks = wttasks.as<int4>();
    d.n_tasks = n_tasks;
    d.wt_perm = wtperm.as<uint16_t>();
    d.wt_heavy = wtheavy.as<int4>();
    d.wt_slot_heavy = wtslotheavy.as<int>();
    d.wt_heavy_cnt = sc.heavy_cnt.as<unsigned>();
    d.n_heavy = n_heavy;
    d.n_slots = n_slots;
    d.wt_part = sc.part_wt.as<cplx<R>>();
    d.Gt = sc.Gt.as<cplx<R>>();
    d.Gth = sc.Gth.as<cplx<R>>();
    d.H = sc.H.as<cplx<R>>();
    d.g = sc.g.as<cplx<R>>();
    d.s = sc.s.as<cplx<R>>();
    d.K = sc.K.as<cplx<R>>();
    d.gram = TaskSpmv<R>{gram.ent.as<WtEnt<R>>(), gram.tasks.as<int4>(), gram.n_tasks, gram.perm.as<uint16_t>(),
                         gram.heavy.as<int4>(), gram.slot_heavy.as<int>(), sc.heavy_cnt_gram.as<unsigned>(),
                         gram.n_heavy, gram.n_slots, sc.part_gram.as<cplx<R>>()};
    // the folded W^T shares the split-block partials / tickets of W^T (never in flight together)
    d.wth = TaskSpmv<R>{herm.ent.as<WtEnt<R>>(), herm.tasks.as<int4>(), herm.n_tasks, herm.perm.as<uint16_t>(),
                        herm.heavy.as<int4>(), herm.slot_heavy.as<int>(), sc.heavy_cnt.as<unsigned>(),
                        herm.n_heavy, herm.n_slots, sc.part_wt.as<cplx<R>>()};
    d.herm_in = d.herm_out = 0;
    return d;
  }

  // split-block partial slots / tickets per slice, shared by W^T and its Hermitian fold
  size_t wt_slots_cap() const { return static_cast<size_t>(std::max({n_slots, herm.n_slots, sym.n_slots, 1})); }
  size_t wt_heavy_cap() const { return static_cast<size_t>(std::max({n_heavy, herm.n_heavy, sym.n_heavy, 1})); }

  void ensure_batch(int B) {
    Scratch& sc = W().sc;
    if (B <= sc.cap) return;
    const size_t m = g.m, n = g.n, cz = 2 * rsz;
    sc.H.ensure(B * m * n * cz);
    sc.g.ensure(B * m * m * cz);
    sc.Gt.ensure(B * m * m * cz);
    CK(cudaMemset(sc.Gt.p, 0, B * m * m * cz));  // untouched spread-grid nodes stay zero
    if (herm_ok()) {  // the fold touches nodes W^T does not: a grid of its own keeps both zero-clean
      sc.Gth.ensure(B * m * m * cz);  // slice stride m^2 like Gt; rows [0, m/2] used
      CK(cudaMemset(sc.Gth.p, 0, B * m * m * cz));
    }
    sc.part_wt.ensure(static_cast<size_t>(B) * wt_slots_cap() * 32 * cz);
    sc.heavy_cnt.ensure(sizeof(unsigned) * static_cast<size_t>(B) * wt_heavy_cap());
    CK(cudaMemset(sc.heavy_cnt.p, 0, sizeof(unsigned) * static_cast<size_t>(B) * wt_heavy_cap()));
    if (fused()) {
      sc.part_gram.ensure(static_cast<size_t>(B) * std::max(gram.n_slots, 1) * 32 * cz);
      const size_t hb = sizeof(unsigned) * static_cast<size_t>(B) * std::max(gram.n_heavy, 1);
      sc.heavy_cnt_gram.ensure(hb);
      CK(cudaMemset(sc.heavy_cnt_gram.p, 0, hb));
    }
    sc.s.ensure(B * s_len() * cz);
    sc.K.ensure(B * n * m * cz);
    sc.sc.ensure(sizeof(SliceScalars) * B);
    CK(cudaMemset(sc.sc.p, 0, sizeof(SliceScalars) * B));
    sc.part.ensure(sizeof(double) * static_cast<size_t>(B) * MAX_PART_BLOCKS * 2);
    const size_t vl = static_cast<size_t>(B) * n * n * rsz;
    for (auto* v : {&sc.r, &sc.p0, &sc.p1, &sc.ap, &sc.x, &sc.rhs, &sc.fid, &sc.mu0, &sc.mu1, &sc.bx0, &sc.bx1,
                    &sc.by0, &sc.by1, &sc.nred, &sc.zero, &sc.u2})
      v->ensure(vl);
    CK(cudaMemset(sc.zero.p, 0, vl));
    sc.upd_log.ensure(sizeof(double) * static_cast<size_t>(B) * kMaxLoggedIters);
    sc.rel_log.ensure(sizeof(double) * static_cast<size_t>(B) * kMaxLoggedIters);
    sc.cap = B;
    clear_graphs();  // buffers moved
  }

  // grids of lane k >= 1 (the apply path only: no solver vectors or scalars)
  void ensure_lane(int k, int B) {
    Scratch& ln = W().lanes[k - 1];
    if (B <= ln.cap) return;
    const size_t m = g.m, n = g.n, cz = 2 * rsz;
    ln.H.ensure(B * m * n * cz);
    ln.g.ensure(B * m * m * cz);
    ln.Gt.ensure(B * m * m * cz);
    CK(cudaMemset(ln.Gt.p, 0, B * m * m * cz));
    if (herm_ok()) {
      ln.Gth.ensure(B * m * m * cz);
      CK(cudaMemset(ln.Gth.p, 0, B * m * m * cz));
    }
    ln.part_wt.ensure(static_cast<size_t>(B) * wt_slots_cap() * 32 * cz);
    ln.heavy_cnt.ensure(sizeof(unsigned) * static_cast<size_t>(B) * wt_heavy_cap());
    CK(cudaMemset(ln.heavy_cnt.p, 0, sizeof(unsigned) * static_cast<size_t>(B) * wt_heavy_cap()));
    if (fused()) {
      ln.part_gram.ensure(static_cast<size_t>(B) * std::max(gram.n_slots, 1) * 32 * cz);
      const size_t hb = sizeof(unsigned) * static_cast<size_t>(B) * std::max(gram.n_heavy, 1);
      ln.heavy_cnt_gram.ensure(hb);
      CK(cudaMemset(ln.heavy_cnt_gram.p, 0, hb));
    }
    ln.s.ensure(B * s_len() * cz);
    ln.K.ensure(B * n * m * cz);
    ln.cap = B;
    clear_graphs();
  }

  Reduce red() {
    Scratch& sc = W().sc;
    return Reduce{sc.sc.as<SliceScalars>(), sc.part.as<double>()};
  }
  SliceScalars* scal() { return W().sc.sc.as<SliceScalars>(); }
};

namespace tomo_b200 {
namespace {
struct LeaseRec {
  const tomo_op* op;
  Workspace* ws;
  int depth;
};
thread_local std::vector<LeaseRec> tl_leases;

// Leases one of the op's workspaces to the calling thread for one API call on `st`. Preference:
// an idle workspace last used on the same stream (its graphs are warm and stream order already
// serialises it), then an idle one whose last call has completed, then a new one (up to
// kMaxWorkspaces), then the least recently used idle one; otherwise wait. A workspace last used on another stream is ordered after that stream's work
// with its `done` event, so device buffers are never shared by two in-flight calls. Nested
// entries on the same thread reuse the outer lease.
class Lease {
 public:
  Lease(tomo_op* op, cudaStream_t st) : op_(op), st_(st) {
    for (auto& r : tl_leases)
      if (r.op == op) {
        ++r.depth;
        nested_ = true;
        return;
      }
    // Under stream capture (the caller records our launches into its own graph) no event may be
    // queried, recorded or waited on: the capture gets a workspace of its own, reserved for that
    // stream, and ordering the graph's replays is the caller's business.
    cudaStreamCaptureStatus cst = cudaStreamCaptureStatusNone;
    if (st && cudaStreamIsCapturing(st, &cst) == cudaSuccess && cst == cudaStreamCaptureStatusActive)
      capturing_ = true;
    std::unique_lock<std::mutex> lk(op->ws_mu);
    for (;;) {
      ws_ = nullptr;
      for (auto& w : op->pool)  // 1. idle, last used on this stream: warm graphs, no wait
        if (!w->busy && w->last_stream == st) {
          ws_ = w.get();
          break;
        }
      if (!ws_ && !capturing_)
        for (auto& w : op->pool)  // 2. idle and its last call has finished on the device
          if (!w->busy && !w->captured && (!w->done || cudaEventQuery(w->done) == cudaSuccess)) {
            ws_ = w.get();
            break;
          }
      if (!ws_ && static_cast<int>(op->pool.size()) < tomo_op::kMaxWorkspaces) {  // 3. a new one
        op->pool.emplace_back(new Workspace());
        ws_ = op->pool.back().get();
      }
      if (!ws_)
        for (auto& w : op->pool)  // 4. least recently used idle one (ordered by its event)
          if (!w->busy && (capturing_ || !w->captured) && (!ws_ || w->last_use < ws_->last_use)) ws_ = w.get();
      if (ws_) break;
      op->ws_cv.wait(lk);
    }
    ws_->busy = true;
    ws_->last_use = ++op->ws_clock;
    if (capturing_) ws_->captured = true;
    lk.unlock();
    if (!capturing_ && ws_->done && ws_->last_stream != st) {
      const cudaError_t e = cudaStreamWaitEvent(st, ws_->done, 0);
      if (e != cudaSuccess) {
        release();
        throw CudaError(std::string("workspace lease: ") + cudaGetErrorString(e));
      }
    }
    tl_leases.push_back({op, ws_, 1});
  }
  ~Lease() {
    if (nested_) {
      for (auto& r : tl_leases)
        if (r.op == op_) --r.depth;
      return;
    }
    tl_leases.pop_back();
    if (!capturing_) {
      if (!ws_->done) cudaEventCreateWithFlags(&ws_->done, cudaEventDisableTiming);
      if (ws_->done) cudaEventRecord(ws_->done, st_);
    }
    ws_->last_stream = st_;
    release();
  }
  Lease(const Lease&) = delete;
  Lease& operator=(const Lease&) = delete;

 private:
  void release() {
    {
      std::lock_guard<std::mutex> lk(op_->ws_mu);
      ws_->busy = false;
    }
    op_->ws_cv.notify_all();
  }
  tomo_op* op_;
  cudaStream_t st_;
  Workspace* ws_ = nullptr;
  bool nested_ = false;
  bool capturing_ = false;
};
}  // namespace
}  // namespace tomo_b200

Workspace& tomo_op::W() const {
  for (auto it = tl_leases.rbegin(); it != tl_leases.rend(); ++it)
    if (it->op == this) return *it->ws;
  throw std::logic_error("libtomo_b200: op scratch used outside a workspace lease");
}

namespace tomo_b200 {
namespace {

// ------------------------------------------------------------------------------------------
// Operator construction: W as SELL-32 ELL (row j, entry e = a*w + b -> node iy*m + ix, value
// wx[a]*wy[b], nufft.cpp:185-200), W^T as SELL-32 over consecutive grid nodes (entries sorted
// by sample index: the exact transpose of the same products, spread nufft.cpp:142-157).
// ------------------------------------------------------------------------------------------
// Task tables of a sparse operator on the grid (W^T, or the Gram for the fused backend), built
// one grid row at a time: per row the nodes are sorted by entry count (descending, stable in
// ix); 32 sorted nodes form a block of L = max count chunks (entries chunk-major, padded with
// weight-0 re-reads of a sample already in cache); blocks with L > max_chunks are split into
// several warp tasks whose partial sums the last task of the block combines.
// The task SpMV loads its entry groups unconditionally (chunks past a task's end belong to the next
// task and gather nothing): every entry stream carries kEntPadChunks zero chunks after its last slot.
constexpr int kEntPadChunks = 16;
template <typename R>
void ent_alloc(Raw& r, int64_t slots) {
  const size_t n = static_cast<size_t>(std::max<int64_t>(slots, 0)) + static_cast<size_t>(kEntPadChunks) * 32;
  r.ensure(sizeof(WtEnt<R>) * n);
  CK(cudaMemset(static_cast<char*>(r.p) + sizeof(WtEnt<R>) * std::max<int64_t>(slots, 0), 0,
                sizeof(WtEnt<R>) * static_cast<size_t>(kEntPadChunks) * 32));
}

template <typename R>
struct TaskBuilder {
  int m, max_chunks;
  std::vector<WtEnt<R>> ent;
  std::vector<int4> tasks, heavy;
  std::vector<int> slot_heavy;
  std::vector<uint16_t> perm;
  std::vector<int> order;
  int slots = 0;
  int64_t chunks = 0, touched = 0;

  TaskBuilder(int m_, int max_chunks_, int64_t nnz_hint)
      : m(m_), max_chunks(max_chunks_), perm(static_cast<size_t>(m_) * m_), order(m_) {
    ent.reserve(static_cast<size_t>(nnz_hint * 1.1) + 32);
  }

  // grid row iy: node ix holds entries [off[ix], off[ix+1]) of (col, val)
  void add_row(int iy, const int64_t* off, const int32_t* col, const R* val) {
    const int bpr = m / 32;
    for (int ix = 0; ix < m; ++ix) {
      order[ix] = ix;
      touched += off[ix + 1] > off[ix];
    }
    std::stable_sort(order.begin(), order.end(),
                     [off](int a, int b) { return off[a + 1] - off[a] > off[b + 1] - off[b]; });
    for (int k = 0; k < m; ++k) perm[static_cast<int64_t>(iy) * m + k] = static_cast<uint16_t>(order[k]);
    for (int kb = 0; kb < bpr; ++kb) {
      const int first = order[kb * 32];
      const int Lb = static_cast<int>(off[first + 1] - off[first]);
      if (!Lb) continue;
      const int64_t c0 = chunks;
      chunks += Lb;
      if (chunks > (int64_t(1) << 31) - 1) throw ConfigError("sparse operator too large for 32-bit chunk indices");
      ent.resize(static_cast<size_t>(chunks) * 32);
      for (int l = 0; l < 32; ++l) {
        const int ix = order[kb * 32 + l];
        const int c = static_cast<int>(off[ix + 1] - off[ix]);
        int lastj = c > 0 ? col[off[ix]] : col[off[first]];
        for (int k = 0; k < Lb; ++k) {
          WtEnt<R> e{};
          if (k < c) {
            lastj = col[off[ix] + k];
            e.j = lastj;
            e.w = val[off[ix] + k];
          } else {
            e.j = lastj;  // padding: re-read an input already in cache, weight 0
            e.w = R(0);
          }
          ent[(static_cast<size_t>(c0) + k) * 32 + l] = e;
        }
      }
      const int bk = iy * bpr + kb;
      if (Lb <= max_chunks) {
        tasks.push_back(make_int4(bk, static_cast<int>(c0), Lb, -1));
      } else {
        const int ns = (Lb + max_chunks - 1) / max_chunks;
        heavy.push_back(make_int4(bk, slots, ns, 0));
        for (int k = 0; k < ns; ++k) slot_heavy.push_back(static_cast<int>(heavy.size()) - 1);
        for (int k = 0; k < ns; ++k) {
          const int cc = k * max_chunks;
          tasks.push_back(make_int4(bk, static_cast<int>(c0) + cc, std::min(max_chunks, Lb - cc), slots++));
        }
      }
    }
  }

  void finish() {
    // longest tasks first (they are launched first and overlap the rest)
    if (!wt_row_order(m))
      std::stable_sort(tasks.begin(), tasks.end(), [](const int4& a, const int4& b) { return a.z > b.z; });
    if (ent.empty()) ent.resize(1);
  }

  void upload(Raw& dent, Raw& dtasks, Raw& dperm, Raw& dheavy, Raw& dslot) const {
    std::vector<WtEnt<R>> padded(ent);
    padded.resize(ent.size() + static_cast<size_t>(kEntPadChunks) * 32, WtEnt<R>{});  // zero tail (see ent_alloc)
    dent.upload(padded);
    dtasks.upload(tasks.empty() ? std::vector<int4>(1) : tasks);
    dperm.upload(perm);
    dheavy.upload(heavy.empty() ? std::vector<int4>(1) : heavy);
    dslot.upload(slot_heavy.empty() ? std::vector<int>(1) : slot_heavy);
  }
};

// Gram W^T W of the spreading operator on the (transposed) grid, build_btb
// (normal_ops.cpp:53-173): entry (u, v) = sum_j W[j][u] W[j][v]; row u reaches the nodes within
// w-1 per axis (band 2w-1). Accumulated in fp64 with a dense band per node over blocks of grid
// rows, samples in ascending order and the reference's product association
// (wx[a]wx[a2]) * (wy[b]wy[b2]), exact zeros dropped. Emits one grid row iy at a time:
// sink(iy, roff[m+1], col (node iy'*m+ix'), val) with node ix's entries at [roff[ix], roff[ix+1]).
template <typename Sink>
void gram_rows(const Geom& g, const Plan& pl, Sink&& sink) {
  const int m = g.m, w = g.w, band = 2 * w - 1, band2 = band * band;
  const int64_t lines_budget = std::max<int64_t>(1, (int64_t(128) << 20) / (static_cast<int64_t>(m) * band2 * 8));
  const int lines = static_cast<int>(std::min<int64_t>(lines_budget, m));
  // samples bucketed by the first grid row of their window (ascending j within a bucket)
  std::vector<int> iy0(g.P), ix0(g.P);
  std::vector<int64_t> boff(m + 1, 0);
  for (int64_t j = 0; j < g.P; ++j) {
    iy0[j] = wrapi(pl.mjy[j] + g.lo, m);
    ix0[j] = wrapi(pl.mjx[j] + g.lo, m);
    boff[iy0[j] + 1]++;
  }
  for (int r = 0; r < m; ++r) boff[r + 1] += boff[r];
  std::vector<int> bucket(g.P);
  {
    std::vector<int64_t> fp(boff.begin(), boff.end() - 1);
    for (int64_t j = 0; j < g.P; ++j) bucket[fp[iy0[j]]++] = static_cast<int>(j);
  }
  std::vector<double> acc(static_cast<size_t>(lines) * m * band2);
  std::vector<double> px(static_cast<size_t>(w) * w), py(static_cast<size_t>(w) * w);
  std::vector<int> list;
  std::vector<int64_t> roff(m + 1);
  std::vector<int32_t> rcol;
  std::vector<double> rval;
  rcol.reserve(static_cast<size_t>(m) * band2);
  rval.reserve(static_cast<size_t>(m) * band2);
  for (int y0 = 0; y0 < m; y0 += lines) {
    const int y1 = std::min(m, y0 + lines);
    std::fill(acc.begin(), acc.begin() + static_cast<size_t>(y1 - y0) * m * band2, 0.0);
    // samples whose window rows iy0..iy0+w-1 (mod m) meet [y0, y1)
    list.clear();
    if (y1 - y0 + w - 1 >= m) {
      for (int64_t j = 0; j < g.P; ++j) list.push_back(static_cast<int>(j));
    } else {
      for (int r = y0 - w + 1; r < y1; ++r) {
        const int rr = wrapi(r, m);
        for (int64_t k = boff[rr]; k < boff[rr + 1]; ++k) list.push_back(bucket[k]);
      }
      std::sort(list.begin(), list.end());
    }
    for (int j : list) {
      const double* wxj = pl.wx.data() + static_cast<size_t>(j) * w;
      const double* wyj = pl.wy.data() + static_cast<size_t>(j) * w;
      for (int a = 0; a < w; ++a)
        for (int a2 = 0; a2 < w; ++a2) px[a * w + a2] = wxj[a] * wxj[a2];
      for (int b = 0; b < w; ++b)
        for (int b2 = 0; b2 < w; ++b2) py[b * w + b2] = wyj[b] * wyj[b2];
      for (int b = 0; b < w; ++b) {
        const int iy = wrapi(iy0[j] + b, m);
        if (iy < y0 || iy >= y1) continue;
        for (int a = 0; a < w; ++a) {
          const int ix = wrapi(ix0[j] + a, m);
          double* cell = acc.data() + (static_cast<size_t>(iy - y0) * m + ix) * band2;
          for (int b2 = 0; b2 < w; ++b2) {
            const double vy = py[b * w + b2];
            double* dst = cell + static_cast<size_t>(b2 - b + w - 1) * band + (w - 1 - a);
            const double* pxa = px.data() + a * w;
            for (int a2 = 0; a2 < w; ++a2) dst[a2] += pxa[a2] * vy;
          }
        }
      }
    }
    for (int iy = y0; iy < y1; ++iy) {
      rcol.clear();
      rval.clear();
      roff[0] = 0;
      for (int ix = 0; ix < m; ++ix) {
        const double* cell = acc.data() + (static_cast<size_t>(iy - y0) * m + ix) * band2;
        for (int dy = 0; dy < band; ++dy) {
          const int cy = wrapi(iy + dy - (w - 1), m);
          for (int dx = 0; dx < band; ++dx) {
            const double v = cell[dy * band + dx];
            if (v != 0.0) {
              rcol.push_back(cy * m + wrapi(ix + dx - (w - 1), m));
              rval.push_back(v);
            }
          }
        }
        roff[ix + 1] = static_cast<int64_t>(rcol.size());
      }
      sink(iy, roff.data(), rcol.data(), rval.data());
    }
  }
}

template <typename R>
void gram_upload(tomo_op* op, TaskBuilder<R>& tb, int64_t nnz) {
  tb.finish();
  TaskSet& ts = op->gram;
  ts.n_tasks = static_cast<int>(tb.tasks.size());
  ts.n_heavy = static_cast<int>(tb.heavy.size());
  ts.n_slots = tb.slots;
  ts.slots = tb.chunks * 32;
  ts.nnz = nnz;
  ts.bytes = ts.slots * static_cast<int64_t>(sizeof(WtEnt<R>)) + static_cast<int64_t>(ts.n_tasks) * 16 +
             static_cast<int64_t>(op->g.m) * op->g.m * 2;
  tb.upload(ts.ent, ts.tasks, ts.perm, ts.heavy, ts.slot_heavy);
}

template <typename R>
void build_gram(tomo_op* op, const Plan& pl) {
  const Geom& g = op->g;
  const int m = g.m, band = 2 * g.w - 1, band2 = band * band;
  const int64_t cap = op->desc.mem_cap_bytes > 0 ? op->desc.mem_cap_bytes : (int64_t(8) << 30);
  const int64_t est = op->wt_rows * static_cast<int64_t>(band2) * 16;
  if (est > cap)
    throw ConfigError("build_btb: estimated " + std::to_string(est >> 20) +
                      " MiB exceeds cap; raise the cap or use a smaller m_sp");
  if (ab_knob("TOMO_BUILD") != "host") {  // on the device (opbuild.cu), same tables
    std::vector<int> base(g.P);
    for (int64_t j = 0; j < g.P; ++j)
      base[j] = wrapi(pl.mjx[j] + g.lo, m) | (wrapi(pl.mjy[j] + g.lo, m) << 16);
    GpuBuildSizes sz{};
    int64_t nnz = 0;
    GpuBuild* raw = gpu_build_gram_begin<R>(m, g.w, g.P, base.data(), pl.wx.data(), pl.wy.data(), 0, &sz, &nnz);
    if (raw) {
      std::unique_ptr<GpuBuild, void (*)(GpuBuild*)> gb(raw, gpu_build_free);
      TaskSet& ts = op->gram;
      ts.n_tasks = sz.n_tasks;
      ts.n_heavy = sz.n_heavy;
      ts.n_slots = sz.n_slots;
      ts.slots = sz.chunks * 32;
      ts.nnz = nnz;
      ts.bytes = ts.slots * static_cast<int64_t>(sizeof(WtEnt<R>)) + static_cast<int64_t>(ts.n_tasks) * 16 +
                 static_cast<int64_t>(m) * m * 2;
      ent_alloc<R>(ts.ent, ts.slots);
      ts.tasks.ensure(sizeof(int4) * std::max(ts.n_tasks, 1));
      ts.perm.ensure(sizeof(uint16_t) * static_cast<size_t>(m) * m);
      ts.heavy.ensure(sizeof(int4) * std::max(ts.n_heavy, 1));
      ts.slot_heavy.ensure(sizeof(int) * std::max(ts.n_slots, 1));
      gpu_build_finish<R>(gb.get(), ts.ent.as<WtEnt<R>>(), ts.tasks.as<int4>(), ts.perm.as<uint16_t>(),
                          ts.heavy.as<int4>(), ts.slot_heavy.as<int>(), 0);
      return;
    }
  }
  TaskBuilder<R> tb(m, wt_max_chunks(), op->wt_rows * band2);
  std::vector<R> rv;
  int64_t nnz = 0;
  gram_rows(g, pl, [&](int iy, const int64_t* roff, const int32_t* rcol, const double* rval) {
    rv.assign(rval, rval + roff[m]);
    tb.add_row(iy, roff, rcol, rv.data());
    nnz += roff[m];
  });
  gram_upload<R>(op, tb, nnz);
}

// Reference cache provenance (bench.cpp:78-84 meta_matches): n, m_sp, tau, angle count, r.
void check_tspm_meta(const tomo_op* op, const TspmFile& t, bool gram) {
  const Geom& g = op->g;
  if (g.lo != -g.hi) throw ConfigError("TOMOSPM1: the reference format needs a symmetric window [-m_sp, m_sp]");
  if (g.nb != g.n || g.R != 2) throw ConfigError("TOMOSPM1: the reference format has n_b = n and R = 2");
  if (op->sharded()) throw ConfigError("TOMOSPM1: operators are whole-geometry (not angle shards)");
  const TspmMeta& mt = t.meta;
  if (mt.n != g.n || mt.m_sp != g.hi || mt.tau != g.tau || mt.angle_count != g.A || (gram ? mt.r != 0 : mt.r < 1))
    throw ConfigError("TOMOSPM1: cache metadata mismatch (n, m_sp, tau, angle count or r)");
  const int64_t side = gram ? static_cast<int64_t>(g.m) * g.m : static_cast<int64_t>(g.n) * g.n;
  if (t.rows != side || t.cols != side) throw ConfigError("TOMOSPM1: operator size does not match the geometry");
}

// Gram from a reference cache file: row tx*m+ty of the reference layout is node ty*m+tx here.
template <typename R>
void gram_from_tspm(tomo_op* op, const TspmFile& t) {
  check_tspm_meta(op, t, true);
  const int m = op->g.m;
  TaskBuilder<R> tb(m, wt_max_chunks(), t.nnz());
  std::vector<int64_t> roff(m + 1);
  std::vector<int32_t> rcol;
  std::vector<R> rval;
  for (int iy = 0; iy < m; ++iy) {
    rcol.clear();
    rval.clear();
    roff[0] = 0;
    for (int ix = 0; ix < m; ++ix) {
      const int64_t r = static_cast<int64_t>(ix) * m + iy;
      for (int64_t k = t.off[r]; k < t.off[r + 1]; ++k) {
        const int c = t.col[k];
        rcol.push_back((c % m) * m + c / m);
        rval.push_back(static_cast<R>(t.val[k]));
      }
      roff[ix + 1] = static_cast<int64_t>(rcol.size());
    }
    tb.add_row(iy, roff.data(), rcol.data(), rval.data());
  }
  gram_upload<R>(op, tb, t.nnz());
}

// The Gram in the reference's CSR layout (row tx*m+ty, columns ascending), fp64, for save_sparse.
TspmFile gram_to_tspm(const tomo_op* op) {
  const Geom& g = op->g;
  const int m = g.m;
  const int64_t G = static_cast<int64_t>(m) * m;
  const Plan pl = make_plan(g);
  // node lists in this layout (iy-major), then re-emitted ix-major with sorted columns
  std::vector<int64_t> noff(G + 1, 0);
  std::vector<int32_t> col;
  std::vector<double> val;
  gram_rows(g, pl, [&](int iy, const int64_t* roff, const int32_t* rcol, const double* rval) {
    const int64_t base = static_cast<int64_t>(col.size());
    for (int ix = 0; ix < m; ++ix) noff[static_cast<int64_t>(iy) * m + ix + 1] = base + roff[ix + 1];
    for (int64_t k = 0; k < roff[m]; ++k) {
      const int c = rcol[k];
      col.push_back((c % m) * m + c / m);
      val.push_back(rval[k]);
    }
  });
  TspmFile t;
  t.rows = t.cols = G;
  t.symmetric = true;
  t.off.reserve(G + 1);
  t.off.push_back(0);
  t.col.reserve(col.size());
  t.val.reserve(val.size());
  std::vector<std::pair<int32_t, double>> row;
  for (int tx = 0; tx < m; ++tx)
    for (int ty = 0; ty < m; ++ty) {
      const int64_t node = static_cast<int64_t>(ty) * m + tx;
      row.clear();
      for (int64_t k = noff[node]; k < noff[node + 1]; ++k) row.emplace_back(col[k], val[k]);
      std::sort(row.begin(), row.end(), [](const auto& a, const auto& b) { return a.first < b.first; });
      for (const auto& e : row) {
        t.col.push_back(e.first);
        t.val.push_back(e.second);
      }
      t.off.push_back(static_cast<int64_t>(t.val.size()));
    }
  return t;
}

// Host build of W (separable) and W^T (fp64 plan, the reference's recurrence); the device
// build (build_w_gpu) produces the same tables and is the default.
template <typename R>
void build_w_host(tomo_op* op) {
  const Geom& g = op->g;
  const Plan pl = make_plan(g);
  const int w = g.w, w2 = w * w;
  const int m = g.m;
  // entries of row j in the reference's loop order (a outer, b inner), nufft.cpp:142-157
  std::vector<int32_t> ent_node(static_cast<size_t>(g.P) * w2);
  std::vector<double> ent_val(ent_node.size());
  std::vector<int> cnt(static_cast<size_t>(m) * m, 0);
  for (int64_t j = 0; j < g.P; ++j) {
    const double* wx = pl.wx.data() + j * w;
    const double* wy = pl.wy.data() + j * w;
    for (int a = 0; a < w; ++a) {
      const int ix = wrapi(pl.mjx[j] + g.lo + a, m);
      for (int b = 0; b < w; ++b) {
        const int iy = wrapi(pl.mjy[j] + g.lo + b, m);
        const size_t e = static_cast<size_t>(j) * w2 + a * w + b;
        ent_node[e] = iy * m + ix;
        ent_val[e] = wx[a] * wy[b];
        cnt[static_cast<size_t>(iy) * m + ix]++;
      }
    }
  }

  // W^T: per grid row, nodes sorted by entry count (descending, stable in ix); 32 sorted nodes
  // form a block of L = max count chunks; entries chunk-major within the block; blocks with
  // L > kWtMaxChunks are split into several tasks whose partials a fix-up kernel sums.
  const int64_t G = static_cast<int64_t>(m) * m;
  std::vector<int64_t> off(G + 1, 0);
  for (int64_t i = 0; i < G; ++i) off[i + 1] = off[i] + cnt[i];
  std::vector<int32_t> tj(off[G]);
  std::vector<R> tv(off[G]);
  std::vector<int64_t> fillp(off.begin(), off.end() - 1);
  for (int64_t j = 0; j < g.P; ++j) {
    for (int e = 0; e < w2; ++e) {
      const size_t o = static_cast<size_t>(j) * w2 + e;
      const int64_t k = fillp[ent_node[o]]++;
      tj[k] = static_cast<int32_t>(j);
      tv[k] = static_cast<R>(ent_val[o]);
    }
  }
  TaskBuilder<R> tb(m, wt_max_chunks(), off[G]);
  for (int iy = 0; iy < m; ++iy) tb.add_row(iy, off.data() + static_cast<int64_t>(iy) * m, tj.data(), tv.data());
  tb.finish();
  op->wt_rows = tb.touched;
  op->wt_slots = tb.chunks * 32;
  op->n_tasks = static_cast<int>(tb.tasks.size());
  op->n_heavy = static_cast<int>(tb.heavy.size());
  op->n_slots = tb.slots;

  // separable storage of the same rows: base node + the two factor vectors (SoA)
  std::vector<int> wbase(op->Ppad, 0);
  std::vector<R> wxs(static_cast<size_t>(w) * op->Ppad, R(0)), wys(static_cast<size_t>(w) * op->Ppad, R(0));
  for (int64_t j = 0; j < g.P; ++j) {
    const int ix0 = wrapi(pl.mjx[j] + g.lo, m), iy0 = wrapi(pl.mjy[j] + g.lo, m);
    wbase[j] = ix0 | (iy0 << 16);
    for (int a = 0; a < w; ++a) {
      wxs[static_cast<size_t>(a) * op->Ppad + j] = static_cast<R>(pl.wx[j * w + a]);
      wys[static_cast<size_t>(a) * op->Ppad + j] = static_cast<R>(pl.wy[j * w + a]);
    }
  }
  op->wbase.upload(wbase);
  op->wxs.upload(wxs);
  op->wys.upload(wys);
  tb.upload(op->wtent, op->wttasks, op->wtperm, op->wtheavy, op->wtslotheavy);
}

// Device build of the separable W and of W^T (opbuild.cu): same tables as build_w_host.
template <typename R>
void build_w_gpu(tomo_op* op) {
  const Geom& g = op->g;
  const int w = g.w, m = g.m;
  BuildArgs a{m, g.nb, g.lo, g.hi, w, g.P, op->Ppad, g.tau};
  std::vector<double> cs;
  for (int k = g.a0; k < g.a1; ++k) {
    cs.push_back(std::cos(g.angles[k]));
    cs.push_back(std::sin(g.angles[k]));
  }
  const double big_m = m / 2.0;
  std::vector<double> e3(w);
  for (int l = g.lo; l <= g.hi; ++l) e3[l - g.lo] = std::exp(-(M_PI * l / big_m) * (M_PI * l / big_m) / (4.0 * g.tau));
  op->wbase.ensure(sizeof(int) * op->Ppad);
  op->wxs.ensure(sizeof(R) * w * op->Ppad);
  op->wys.ensure(sizeof(R) * w * op->Ppad);
  GpuBuildSizes sz{};
  std::unique_ptr<GpuBuild, void (*)(GpuBuild*)> b(
      gpu_build_begin<R>(a, cs.data(), e3.data(), op->wbase.as<int>(), op->wxs.as<R>(), op->wys.as<R>(), 0, &sz),
      gpu_build_free);
  op->wt_rows = sz.touched;
  op->wt_slots = sz.chunks * 32;
  op->n_tasks = sz.n_tasks;
  op->n_heavy = sz.n_heavy;
  op->n_slots = sz.n_slots;
  ent_alloc<R>(op->wtent, op->wt_slots);
  op->wttasks.ensure(sizeof(int4) * std::max(sz.n_tasks, 1));
  op->wtperm.ensure(sizeof(uint16_t) * static_cast<size_t>(m) * m);
  op->wtheavy.ensure(sizeof(int4) * std::max(sz.n_heavy, 1));
  op->wtslotheavy.ensure(sizeof(int) * std::max(sz.n_slots, 1));
  gpu_build_finish<R>(b.get(), op->wtent.as<WtEnt<R>>(), op->wttasks.as<int4>(), op->wtperm.as<uint16_t>(),
                      op->wtheavy.as<int4>(), op->wtslotheavy.as<int>(), 0);
  // the Hermitian fold of the same W^T for real-part outputs (real subspace)
  if (ab_knob("TOMO_HERM") == "0") return;
  GpuBuildSizes hz{};
  std::unique_ptr<GpuBuild, void (*)(GpuBuild*)> hb(gpu_build_fold<R>(b.get(), 0, &hz), gpu_build_free);
  TaskSet& ts = op->herm;
  ts.nnz = hz.nnz;
  ts.touched = hz.touched;
  ts.n_tasks = hz.n_tasks;
  ts.n_heavy = hz.n_heavy;
  ts.n_slots = hz.n_slots;
  ts.slots = hz.chunks * 32;
  ent_alloc<R>(ts.ent, ts.slots);
  ts.tasks.ensure(sizeof(int4) * std::max(ts.n_tasks, 1));
  ts.perm.ensure(sizeof(uint16_t) * static_cast<size_t>(m / 2 + 1) * m);
  ts.heavy.ensure(sizeof(int4) * std::max(ts.n_heavy, 1));
  ts.slot_heavy.ensure(sizeof(int) * std::max(ts.n_slots, 1));
  gpu_build_finish<R>(hb.get(), ts.ent.as<WtEnt<R>>(), ts.tasks.as<int4>(), ts.perm.as<uint16_t>(),
                      ts.heavy.as<int4>(), ts.slot_heavy.as<int>(), 0);
  // mirror pairs of the samples: the primaries' fold (half the entries) for the normal operator
  if (ab_knob("TOMO_SYM") == "0" || g.P <= 0) return;
  op->pairs.ensure(sizeof(int) * g.P);
  op->n_paired = gpu_find_pairs<R>(a, op->wbase.as<int>(), op->wxs.as<R>(), op->wys.as<R>(), op->pairs.as<int>(), 0);
  // worth its two extra tables only when most samples pair up (the reference's symmetric window
  // [-m_sp, m_sp] around floor(x / h) pairs nothing but the few samples that sit on a grid line)
  if (op->n_paired * 2 < g.P) {
    op->n_paired = 0;
    return;
  }
  const int mode = g.lo == 1 - g.hi ? 1 : 2;
  if (mode == 2 && ab_knob("TOMO_SYM") == "1") {  // A/B: mirror-image windows only
    op->n_paired = 0;
    return;
  }
  GpuBuildSizes yz{};
  std::unique_ptr<GpuBuild, void (*)(GpuBuild*)> yb(
      gpu_build_fold<R>(b.get(), 0, &yz, op->pairs.as<int>(), mode == 2 ? op->wbase.as<int>() : nullptr),
      gpu_build_free);
  // the primaries' fold must write every node the full fold writes (they share the half grid
  // buffer, whose untouched nodes stay zero); mirror-image windows guarantee it
  if (yz.touched != hz.touched) {
    op->n_paired = 0;
    return;
  }
  TaskSet& ys = op->sym;
  ys.nnz = yz.nnz;
  ys.touched = yz.touched;
  ys.n_tasks = yz.n_tasks;
  ys.n_heavy = yz.n_heavy;
  ys.n_slots = yz.n_slots;
  ys.slots = yz.chunks * 32;
  ent_alloc<R>(ys.ent, ys.slots);
  ys.tasks.ensure(sizeof(int4) * std::max(ys.n_tasks, 1));
  ys.perm.ensure(sizeof(uint16_t) * static_cast<size_t>(m / 2 + 1) * m);
  ys.heavy.ensure(sizeof(int4) * std::max(ys.n_heavy, 1));
  ys.slot_heavy.ensure(sizeof(int) * std::max(ys.n_slots, 1));
  gpu_build_finish<R>(yb.get(), ys.ent.as<WtEnt<R>>(), ys.tasks.as<int4>(), ys.perm.as<uint16_t>(),
                      ys.heavy.as<int4>(), ys.slot_heavy.as<int>(), 0);
  op->sym_mode = mode;
}

template <typename R>
void build_tables(tomo_op* op) {
  const Geom& g = op->g;
  const int w = g.w, m = g.m;
  op->Ppad = static_cast<int>((g.P + 31) / 32 * 32);
  op->nnz = g.P * w * w;
  // W / W^T are built on the device; TOMO_BUILD=host (with TOMO_AB=1) selects the host build,
  // kept as the reference the device tables are compared with (tests/test_gpu_build.py)
  if (ab_knob("TOMO_BUILD") == "host")
    build_w_host<R>(op);
  else
    build_w_gpu<R>(op);
  // separable W in 16x16 grid-tile order: concurrently running warps gather from nearby nodes
  op->w_sorted = true;
  {
    op->wperm.ensure(sizeof(int) * std::max<int64_t>(g.P, 1));
    gpu_sort_w_tables<R>(m, g.P, op->Ppad, w, op->wbase.as<int>(), op->wxs.as<R>(), op->wys.as<R>(),
                         op->wperm.as<int>(), op->wtent.as<WtEnt<R>>(), op->wt_slots, op->herm.ent.as<WtEnt<R>>(),
                         op->herm.slots, 0);
  }
  if (op->sym.n_tasks > 0 && op->sym_mode == 2) {
    // overlap pairs: entries to positions (pair sums behind the samples), partner positions
    op->ppos.ensure(sizeof(int) * g.P);
    gpu_pair_sigma_setup<R>(g.P, op->wperm.as<int>(), op->pairs.as<int>(), op->sym.ent.as<WtEnt<R>>(), op->sym.slots,
                            op->ppos.as<int>(), 0);
    if (g.lo == -g.hi && w + 1 <= 8 && ab_knob("TOMO_PAIR_W") != "0") {
      // W by units: one thread per mirror pair / unpaired sample over the (w + 1)^2 union window
      // (symmetric windows: the partner's mirrored window is the primary's shifted up by one node)
      int64_t U = 0;
      std::unique_ptr<HalfWBuild, void (*)(HalfWBuild*)> hw(
          gpu_half_w_begin(g.P, op->wperm.as<int>(), op->pairs.as<int>(), 0, &U), gpu_half_w_free);
      op->n_units = U;
      op->Upad = static_cast<int>((U + 31) / 32 * 32);
      op->hbase.ensure(sizeof(int) * op->Upad);
      op->hwx.ensure(sizeof(R) * (w + 1) * op->Upad);
      op->hwy.ensure(sizeof(R) * (w + 1) * op->Upad);
      op->upos.ensure(sizeof(int) * op->Upad);
      op->uppos.ensure(sizeof(int) * op->Upad);
      gpu_pair_w_finish<R>(hw.get(), op->Ppad, op->Upad, w, op->ppos.as<int>(), op->wbase.as<int>(), op->wxs.as<R>(),
                           op->wys.as<R>(), op->hbase.as<int>(), op->hwx.as<R>(), op->hwy.as<R>(),
                           op->upos.as<int>(), op->uppos.as<int>(), 0);
    }
  } else if (op->sym.n_tasks > 0) {
    // the half W (one sample per mirror pair + the unpaired ones, tile order kept); the mirror-pair
    // W^T's entries move from sample indices to the half W's output positions
    int64_t Ph = 0;
    std::unique_ptr<HalfWBuild, void (*)(HalfWBuild*)> hw(
        gpu_half_w_begin(g.P, op->wperm.as<int>(), op->pairs.as<int>(), 0, &Ph), gpu_half_w_free);
    op->Ph = Ph;
    op->Ppad_h = static_cast<int>((Ph + 31) / 32 * 32);
    op->hbase.ensure(sizeof(int) * op->Ppad_h);
    op->hwx.ensure(sizeof(R) * w * op->Ppad_h);
    op->hwy.ensure(sizeof(R) * w * op->Ppad_h);
    gpu_half_w_finish<R>(hw.get(), op->Ppad, op->Ppad_h, w, op->wperm.as<int>(), op->pairs.as<int>(),
                         op->wbase.as<int>(), op->wxs.as<R>(), op->wys.as<R>(), op->hbase.as<int>(),
                         op->hwx.as<R>(), op->hwy.as<R>(), op->sym.ent.as<WtEnt<R>>(), op->sym.slots, 0);
  }
  // deapodisation a[t]/m (nufft.cpp:204-227 with the 1/m per-axis FFT scale folded in)
  std::vector<R> apod(g.n);
  const double root = std::sqrt(M_PI / g.tau);
  for (int t = 0; t < g.n; ++t) {
    const double k = t - g.n / 2;
    apod[t] = static_cast<R>(root * std::exp(k * k * g.tau) / m);
  }
  std::vector<cplx<R>> tw(m);
  for (int k = 0; k < m; ++k) {
    const double ang = -2.0 * M_PI * static_cast<double>(k) / m;
    tw[k].x = static_cast<R>(std::cos(ang));
    tw[k].y = static_cast<R>(std::sin(ang));
  }
  std::vector<cplx<R>> twh(m / 2);
  for (int k = 0; k < m / 2; ++k) {
    const double ang = -2.0 * M_PI * static_cast<double>(k) / (m / 2);
    twh[k].x = static_cast<R>(std::cos(ang));
    twh[k].y = static_cast<R>(std::sin(ang));
  }
  op->apod.upload(apod);
  op->tw.upload(tw);
  op->twh.upload(twh);
  if (op->fused()) {
    if (op->src)
      gram_from_tspm<R>(op, *op->src);
    else
      build_gram<R>(op, make_plan(g));
  }
}

// ------------------------------------------------------------------------------------------
// Pipelines (all device pointers, stream-ordered)
// ------------------------------------------------------------------------------------------
template <typename R>
void allreduce(tomo_op* op, R* buf, size_t count, cudaStream_t st) {
  if (!op->sharded()) return;
  if (op->comm) {
    const ncclResult_t r = ncclAllReduce(buf, buf, count, sizeof(R) == 8 ? ncclFloat64 : ncclFloat32, ncclSum,
                                         op->comm, st);
    if (r != ncclSuccess) throw CudaError(std::string("ncclAllReduce: ") + ncclGetErrorString(r));
  } else if (op->ar_fn) {
    if (op->ar_fn(buf, count, sizeof(R) == 8 ? TOMO_F64 : TOMO_F32, st, op->ar_user) != 0)
      throw CudaError("allreduce hook failed");
  } else {
    throw ConfigError("sharded op needs an all-reduce (tomo_op_attach_nccl / tomo_op_set_allreduce)");
  }
}

// F_NU^* into d.s (the op's internal sample order) or, with ext_out, into an external buffer in
// the reference's sample order.
template <typename R>
void type2(tomo_op* op, int B, const void* in, bool complex_in, const PUpd<R>& pu, cplx<R>* ext_out,
           const SliceScalars* skip, cudaStream_t st) {
  OpDev<R> d = op->dev<R>(B);
  d.herm_in = op->herm_ok() && !complex_in;
  launch_t2_rows<R>(d, B, in, complex_in, pu, st);
  launch_t2_cols<R>(d, B, skip, st);
  if (ext_out) d.w_out_pos = 0;
  launch_w<R>(d, B, d.g, ext_out ? ext_out : d.s, skip, st);
}

// External samples (reference order) -> d.s in the op's internal order.
template <typename R>
cplx<R>* samples_in(tomo_op* op, int B, const cplx<R>* ext, cudaStream_t st) {
  OpDev<R> d = op->dev<R>(B);
  if (op->w_sorted)
    launch_gather_samples<R>(ext, d.s, d.w_perm, B, static_cast<int>(op->g.P), st);
  else if (ext != d.s)
    CK(cudaMemcpyAsync(d.s, ext, sizeof(cplx<R>) * B * op->g.P, cudaMemcpyDeviceToDevice, st));
  return d.s;
}

// F_NU of the samples in d.s (internal order).
template <typename R>
void type1(tomo_op* op, int B, const PbEpi<R>& e, const SliceScalars* skip, cudaStream_t st) {
  OpDev<R> d = op->dev<R>(B);
  d.herm_out = op->herm_ok() && e.mode != PB_COMPLEX;
  if (d.herm_out) d.Gt = d.Gth;
  launch_wt_rows<R>(d, B, skip, st);
  launch_t1_rows<R>(d, B, e, st);
}

template <typename R>
PbEpi<R> plain_epi(int mode, double scale) {
  PbEpi<R> e{};
  e.mode = mode;
  e.scale = static_cast<R>(scale);
  return e;
}

// One normal-operator apply N = F_NU F_NU^* through the five-kernel pipeline:
// P1 (p-update, deapod, pad, row iFFT) -> P2 (column iFFT) -> [W then W^T | Gram W^T W]
// -> PA (pruned column FFT) -> PB (row FFT, crop, deapod, epilogue `e`).
// Direct: apply_normal_direct (normal_ops.cpp:28-30); fused: apply_normal_fused (:175-206).
template <typename R>
void normal_core(tomo_op* op, int B, const void* in, bool complex_in, const PUpd<R>& pu, const PbEpi<R>& e,
                 const SliceScalars* skip, cudaStream_t st) {
  OpDev<R> d = op->dev<R>(B);
  // real image in / real part out: the Hermitian half-grid pipeline (not through the Gram, whose
  // input is the full grid)
  d.herm_in = op->herm_ok() && !op->fused() && !complex_in;
  d.herm_out = op->herm_ok() && !op->fused() && e.mode != PB_COMPLEX;
  if (d.herm_out) d.Gt = d.Gth;
  // real in and real out: W on one sample per mirror pair, the primaries' folded W^T
  if (d.herm_in && d.herm_out && op->sym_ok()) op->use_sym(d);
  launch_t2_rows<R>(d, B, in, complex_in, pu, st);
  launch_t2_cols<R>(d, B, skip, st);
  if (op->fused()) {
    launch_gram<R>(d, B, d.g, d.Gt, skip, st);
    launch_t1_cols_only<R>(d, B, skip, st);
  } else {
    if (d.s_stride == 2 * d.P && op->n_units > 0) {
      launch_w_pair<R>(d, op->pair_w<R>(), B, d.g, d.s, skip, st);  // overlap pairs: W by units, pair sums included
    } else {
      launch_w<R>(d, B, d.g, d.s, skip, st);
      if (d.s_stride == 2 * d.P)  // overlap pairs: the pair sums behind each slice's samples
        launch_pair_sigma<R>(d.s, B, d.P, d.s_stride, op->ppos.as<int>(), st);
    }
    launch_wt_rows<R>(d, B, skip, st);  // W^T + PA (one fused kernel where available)
  }
  launch_t1_rows<R>(d, B, e, st);
}

// Multi-lane execution of a batch of independent slices: the batch is cut into `lanes`
// near-equal sub-batches; sub-batch 0 runs on `st` (lane 0), sub-batch k on the op's lane-k
// stream with lane-k buffers, forked from and joined back into `st` with events (also inside
// CUDA-graph capture). Concurrent lanes overlap the latency-bound passes of one apply with those
// of the others. Measured (bench, applies/s): c3 calls of 2 / 3 / 4 inputs on 2 / 3 / 4 lanes
// 10.8k / 10.9k / 10.7k; c1 calls of 20 inputs on 2 / 4 lanes 49.1k / 53.9k, calls of 12 on 3
// lanes 50.4k. TOMO_LANES=1..4 overrides the default (3). f(b0, nb, stream) runs slices
// [b0, b0 + nb) of the batch.
int lanes_cfg() {
  static const int v = [] {
    const char* e = std::getenv("TOMO_LANES");
    const int k = e && *e ? std::atoi(e) : 3;
    return std::min(std::max(k, 1), static_cast<int>(tomo_op::kMaxLanes));
  }();
  return v;
}

template <typename F>
void run_lanes(tomo_op* op, int batch, cudaStream_t st, F&& f) {
  const int nl = std::min(batch, lanes_cfg());
  if (nl < 2 || op->sharded()) {
    f(0, batch, st);
    return;
  }
  if (!op->W().lane_fork) CK(cudaEventCreateWithFlags(&op->W().lane_fork, cudaEventDisableTiming));
  for (int k = 1; k < nl; ++k)
    if (!op->W().lane_st[k - 1]) {
      CK(cudaStreamCreateWithFlags(&op->W().lane_st[k - 1], cudaStreamNonBlocking));
      CK(cudaEventCreateWithFlags(&op->W().lane_join[k - 1], cudaEventDisableTiming));
    }
  // sub-batch k = [bs(k), bs(k+1)): sizes differ by at most one, larger ones first
  auto bs = [&](int k) { return k * (batch / nl) + std::min(k, batch % nl); };
  op->ensure_batch(bs(1));
  for (int k = 1; k < nl; ++k) op->ensure_lane(k, bs(k + 1) - bs(k));
  CK(cudaEventRecord(op->W().lane_fork, st));
  for (int k = 1; k < nl; ++k) CK(cudaStreamWaitEvent(op->W().lane_st[k - 1], op->W().lane_fork, 0));
  f(0, bs(1), st);
  try {
    for (int k = 1; k < nl; ++k) {
      op->W().cur_lane = k;
      f(bs(k), bs(k + 1) - bs(k), op->W().lane_st[k - 1]);
    }
  } catch (...) {
    op->W().cur_lane = 0;
    throw;
  }
  op->W().cur_lane = 0;
  for (int k = 1; k < nl; ++k) {
    CK(cudaEventRecord(op->W().lane_join[k - 1], op->W().lane_st[k - 1]));
    CK(cudaStreamWaitEvent(st, op->W().lane_join[k - 1], 0));
  }
}

// Re(N u) (or N u complex) for the W/W^T and Gram backends, incl. the cross-rank sum when
// sharded.
template <typename R>
void normal_direct(tomo_op* op, int B, const void* in, bool cplx_io, void* out, cudaStream_t st) {
  PUpd<R> pu{};
  PbEpi<R> e = plain_epi<R>(cplx_io ? PB_COMPLEX : PB_REAL, 1.0);
  if (cplx_io)
    e.out_c = static_cast<cplx<R>*>(out);
  else
    e.out_r = static_cast<R*>(out);
  normal_core<R>(op, B, in, cplx_io, pu, e, nullptr, st);
  allreduce<R>(op, static_cast<R*>(out), static_cast<size_t>(B) * op->L() * (cplx_io ? 2 : 1), st);
}

SysParams sysp(double alpha, double lambda, double shift, double tol) { return SysParams{alpha, lambda, shift, tol}; }

// Chronopoulos-Gear CG for the unsharded W/W^T and Gram backends unless TOMO_CG=std (A/B).
bool cgcg_on() {
  static const bool v = ab_knob("TOMO_CG") != "std";
  return v;
}

// cg_solve (solver.cpp:56-95) for B slices: rhs, x0 -> x (device, B x L each).
template <typename R>
void cg_run(tomo_op* op, int B, const SysParams& s, const R* rhs, const R* x0, R* x, int steps, cudaStream_t st) {
  const int n = op->g.n;
  const int64_t L = op->L();
  Scratch& S = op->W().sc;
  Reduce red = op->red();
  const SliceScalars* skip = op->scal();
  R* r = S.r.as<R>();
  R* p0 = S.p0.as<R>();
  R* p1 = S.p1.as<R>();
  R* ap = S.ap.as<R>();
  if (op->surrogate()) {
    launch_stencil<R>(n, B, op->rad, op->coef, 1, x0, nullptr, p0, r, rhs, x, s, 0, red, st);
    R* cur = p0;
    R* other = p1;
    for (int k = 0; k < steps; ++k) {
      if (k == 0) {
        launch_stencil<R>(n, B, op->rad, op->coef, 0, cur, r, cur, ap, nullptr, nullptr, s, k, red, st);
      } else {
        launch_stencil<R>(n, B, op->rad, op->coef, 0, cur, r, other, ap, nullptr, nullptr, s, k, red, st);
        std::swap(cur, other);
      }
      launch_cg_update<R>(n, B, cur, ap, x, r, s, k, red, st);
    }
    return;
  }
  // W / W^T (or Gram) backend: init r = b - A x0, p = r, x = x0
  const bool shard = op->sharded();
  R* nred = S.nred.as<R>();
  {
    PUpd<R> pu{};
    pu.red = red;
    if (!shard) {
      PbEpi<R> e = plain_epi<R>(PB_CG_INIT, s.alpha);
      e.p = x0;
      e.b = rhs;
      e.ap = r;
      e.p_out = p0;
      e.x_out = x;
      e.sys = s;
      e.step = 0;
      e.red = red;
      normal_core<R>(op, B, x0, false, pu, e, nullptr, st);
    } else {
      PbEpi<R> e = plain_epi<R>(PB_REAL, s.alpha);
      e.out_r = nred;
      normal_core<R>(op, B, x0, false, pu, e, nullptr, st);
      allreduce<R>(op, nred, static_cast<size_t>(B) * L, st);
      launch_cg_epilogue<R>(n, B, 1, nred, x0, rhs, r, p0, x, s, 0, red, st);
    }
  }
  if (cgcg_on() && !shard) {
    // Chronopoulos-Gear CG: each step applies the operator to r (w = A r) with r.w and r.r in
    // the epilogue; the vector update is fused into the next step's first FFT pass, so a step is
    // one apply with one reduction (standard CG: an apply plus an update kernel, two
    // reductions). Same iterates in exact arithmetic; the reference's exits and steps_run are
    // kept (cgcg_finalize). TOMO_CG=std selects the standard two-kernel form.
    R* s_vec = p1;
    for (int k = 0; k < steps; ++k) {
      PUpd<R> pu{};
      pu.enabled = 1;
      pu.cgcg = 1;
      pu.r = r;
      pu.p = p0;
      pu.s = s_vec;
      pu.w = ap;
      pu.x = x;
      pu.step = k;
      pu.red = red;
      PbEpi<R> e = plain_epi<R>(PB_CGCG, s.alpha);
      e.p = r;
      e.ap = ap;
      e.sys = s;
      e.step = k;
      e.red = red;
      normal_core<R>(op, B, r, false, pu, e, skip, st);
    }
    launch_cgcg_final<R>(n, B, ap, p0, s_vec, x, r, s, steps, red, st);
    return;
  }
  for (int k = 0; k < steps; ++k) {
    PUpd<R> pu{};
    pu.enabled = 1;
    pu.r = r;
    pu.p = p0;
    pu.step = k;
    pu.red = red;
    if (!shard) {
      PbEpi<R> e = plain_epi<R>(PB_CG_STEP, s.alpha);
      e.p = p0;
      e.ap = ap;
      e.sys = s;
      e.step = k;
      e.red = red;
      normal_core<R>(op, B, p0, false, pu, e, skip, st);
    } else {
      PbEpi<R> e = plain_epi<R>(PB_REAL, s.alpha);
      e.out_r = nred;
      normal_core<R>(op, B, p0, false, pu, e, skip, st);
      allreduce<R>(op, nred, static_cast<size_t>(B) * L, st);
      launch_cg_epilogue<R>(n, B, 0, nred, p0, nullptr, ap, nullptr, nullptr, s, k, red, st);
    }
    launch_cg_update<R>(n, B, p0, ap, x, r, s, k, red, st);
  }
}

// Back-projection alpha*Re(F_NU f) (solver.cpp:200-213), optionally density weighted.
template <typename R>
void backproject(tomo_op* op, int B, double alpha, bool weighted, const cplx<R>* f, R* out, cudaStream_t st) {
  cplx<R>* s = samples_in<R>(op, B, f, st);
  if (weighted) {
    OpDev<R> d = op->dev<R>(B);
    launch_weight_samples<R>(s, B, static_cast<int>(op->g.P), op->g.nb, d.w_perm, st);
  }
  PbEpi<R> e = plain_epi<R>(PB_REAL, alpha);
  e.out_r = out;
  type1<R>(op, B, e, nullptr, st);
  allreduce<R>(op, out, static_cast<size_t>(B) * op->L(), st);
}

// ---- graph capture of a solver loop -------------------------------------------------------
template <typename F>
void run_graph(tomo_op* op, const std::string& key, cudaStream_t st, F&& body) {
  // A caller all-reduce hook runs on the host (it may synchronize the stream and exchange
  // through the host), so it cannot be captured: such ops run their solver loops eagerly.
  if (op->ar_fn && !op->comm && op->sharded()) {
    body(st);
    return;
  }
  auto it = op->W().graphs.find(key);
  if (it == op->W().graphs.end()) {
    // Capture on a private stream so a legacy default stream (0) can still be used.
    cudaStream_t cs;
    CK(cudaStreamCreateWithFlags(&cs, cudaStreamNonBlocking));
    int64_t count = 0;
    g_capture_count = &count;
    cudaGraph_t graph = nullptr;
    try {
      CK(cudaStreamBeginCapture(cs, cudaStreamCaptureModeThreadLocal));
      body(cs);
      CK(cudaStreamEndCapture(cs, &graph));
    } catch (...) {
      g_capture_count = nullptr;
      cudaGraph_t tmp = nullptr;
      cudaStreamEndCapture(cs, &tmp);
      if (tmp) cudaGraphDestroy(tmp);
      cudaStreamDestroy(cs);
      throw;
    }
    g_capture_count = nullptr;
    GraphEntry ge;
    ge.nodes = count;
    const cudaError_t ie = cudaGraphInstantiate(&ge.exec, graph, 0);
    cudaGraphDestroy(graph);
    cudaStreamDestroy(cs);
    CK(ie);
    it = op->W().graphs.emplace(key, ge).first;
  }
  CK(cudaGraphLaunch(it->second.exec, st));
  g_launches.fetch_add(it->second.nodes, std::memory_order_relaxed);
}

std::string fmtkey(const char* kind, int B, std::initializer_list<double> vals) {
  std::string k = std::string(kind) + ":" + std::to_string(B);
  char buf[64];
  for (double v : vals) {
    std::snprintf(buf, sizeof(buf), ":%.17g", v);
    k += buf;
  }
  return k;
}

// ---- Lanczos sigma (solver.cpp:97-130, 175-192), device ops + host tridiagonal --------------
double tridiag_min(const std::vector<double>& a, const std::vector<double>& b) {
  const int m = static_cast<int>(a.size());
  double lo = 1e300, hi = -1e300;
  for (int i = 0; i < m; ++i) {
    double rad = 0.0;
    if (i > 0) rad += std::fabs(b[i - 1]);
    if (i + 1 < m) rad += std::fabs(b[i]);
    lo = std::min(lo, a[i] - rad);
    hi = std::max(hi, a[i] + rad);
  }
  for (int it = 0; it < 200; ++it) {
    const double mid = 0.5 * (lo + hi);
    if (mid <= lo || mid >= hi) break;
    int cnt = 0;
    double q = 1.0;
    for (int i = 0; i < m; ++i) {
      q = a[i] - mid - (i > 0 ? b[i - 1] * b[i - 1] / q : 0.0);
      if (q == 0.0) q = -1e-300;
      if (q < 0.0) ++cnt;
    }
    if (cnt > 0) hi = mid; else lo = mid;
  }
  return 0.5 * (lo + hi);
}

template <typename R>
double device_dot(tomo_op* op, const R* x, const R* y, cudaStream_t st) {
  launch_dot<R>(op->g.n, 1, x, y, op->red(), st);
  double v = 0.0;
  CK(cudaMemcpyAsync(&v, &op->scal()[0].dot, sizeof(double), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  return v;
}

// make_subproblem's surrogate shift (solver.cpp:175-192) by 40-step Lanczos (lanczos_extreme_ritz,
// :97-130; device applies and dots, host tridiagonal bisection). Without data feedback: the PSD
// floor 1.2 max(0, -lambda_min(alpha T + lambda K'K)); with it: the contraction floor
// 1.2 max(0, lambda_max(alpha F W F* - 2 (alpha T + lambda K'K)) / 2).
template <typename R>
double surrogate_sigma(tomo_op* op, double alpha, double lambda, cudaStream_t st, bool feedback = false) {
  auto key = std::make_pair(alpha, feedback ? -lambda - 1.0 : lambda);  // lambda > 0: distinct keys
  {
    std::lock_guard<std::mutex> lk(op->cache_mu);
    auto it = op->sigma_cache.find(key);
    if (it != op->sigma_cache.end()) return it->second;
  }
  const int n = op->g.n;
  const int64_t L = op->L();
  op->ensure_batch(1);
  Scratch& S = op->W().sc;
  std::mt19937_64 rng(7);
  std::normal_distribution<double> gauss;
  std::vector<double> v(L);
  double nn = 0.0;
  for (auto& e : v) {
    e = gauss(rng);
    nn += e * e;
  }
  nn = std::sqrt(nn);
  std::vector<R> vf(L);
  for (int64_t i = 0; i < L; ++i) vf[i] = static_cast<R>(v[i] / nn);
  R* vcur = S.x.as<R>();
  R* vprev = S.p0.as<R>();
  R* w = S.ap.as<R>();
  R* w2 = S.u2.as<R>();
  CK(cudaMemcpyAsync(vcur, vf.data(), sizeof(R) * L, cudaMemcpyHostToDevice, st));
  CK(cudaMemsetAsync(vprev, 0, sizeof(R) * L, st));
  const SysParams sp = sysp(alpha, lambda, 0.0, 0.0);
  std::vector<double> alphas, betas;
  double beta = 0.0, extreme = 0.0;
  for (int itr = 0; itr < 40; ++itr) {
    if (!feedback) {
      launch_stencil<R>(n, 1, op->rad, op->coef, 2, vcur, nullptr, nullptr, w, nullptr, nullptr, sp, 0, op->red(), st);
    } else {  // w = alpha Re(F W F* v) - 2 (alpha T + lambda K'K) v
      launch_stencil<R>(n, 1, op->rad, op->coef, 2, vcur, nullptr, nullptr, w2, nullptr, nullptr, sp, 0, op->red(), st);
      PUpd<R> pu{};
      type2<R>(op, 1, vcur, false, pu, nullptr, nullptr, st);
      OpDev<R> d = op->dev<R>(1);
      launch_weight_samples<R>(d.s, 1, static_cast<int>(op->g.P), op->g.nb, d.w_perm, st);
      PbEpi<R> e = plain_epi<R>(PB_REAL, 1.0);
      e.out_r = w;
      type1<R>(op, 1, e, nullptr, st);
      launch_axpby<R>(L, alpha, w, -2.0, w2, w, st);
    }
    const double a = device_dot<R>(op, vcur, w, st);
    alphas.push_back(a);
    launch_axpby<R>(L, 1.0, w, -a, vcur, w, st);
    launch_axpby<R>(L, 1.0, w, -beta, vprev, w, st);
    beta = std::sqrt(device_dot<R>(op, w, w, st));
    if (feedback) {  // largest Ritz value: -(smallest of -T)
      std::vector<double> neg(alphas.size());
      for (size_t k = 0; k < alphas.size(); ++k) neg[k] = -alphas[k];
      extreme = -tridiag_min(neg, betas);
    } else {
      extreme = tridiag_min(alphas, betas);
    }
    if (beta < 1e-12) break;
    betas.push_back(beta);
    std::swap(vprev, vcur);                                    // vprev <- v
    launch_axpby<R>(L, 1.0 / beta, w, 0.0, w, vcur, st);       // v <- w / beta
  }
  const double sigma = feedback ? 1.2 * std::max(0.0, 0.5 * extreme) : 1.2 * std::max(0.0, -extreme);
  std::lock_guard<std::mutex> lk(op->cache_mu);
  op->sigma_cache[key] = sigma;
  return sigma;
}

// Surrogate stencil: centre response of the density-weighted normal operator
// (normal_ops.cpp:232-264), computed through the GPU W/W^T path, symmetrised on the host.
template <typename R>
void build_stencil(tomo_op* op, cudaStream_t st) {
  const int n = op->g.n, r = op->desc.surrogate_r;
  if (r < 1 || r > 4 || r >= n / 2) throw ConfigError("build_surrogate: radius out of range (GPU supports 1..4)");
  if (op->sharded()) throw ConfigError("surrogate backend cannot be angle-sharded");
  op->rad = r;
  const int64_t L = op->L();
  op->ensure_batch(1);
  Scratch& S = op->W().sc;
  S.cin.ensure(L * sizeof(cplx<R>));
  S.fout.ensure(L * sizeof(R));
  std::vector<cplx<R>> delta(L);
  for (auto& z : delta) z.x = z.y = R(0);
  delta[static_cast<int64_t>(n / 2) * n + n / 2].x = R(1);
  CK(cudaMemcpyAsync(S.cin.p, delta.data(), sizeof(cplx<R>) * L, cudaMemcpyHostToDevice, st));
  OpDev<R> d = op->dev<R>(1);
  PUpd<R> pu{};
  type2<R>(op, 1, S.cin.p, true, pu, nullptr, nullptr, st);
  launch_weight_samples<R>(d.s, 1, static_cast<int>(op->g.P), op->g.nb, d.w_perm, st);
  PbEpi<R> e = plain_epi<R>(PB_REAL, 1.0);
  e.out_r = S.fout.as<R>();
  type1<R>(op, 1, e, nullptr, st);
  std::vector<R> resp(L);
  CK(cudaMemcpyAsync(resp.data(), S.fout.p, sizeof(R) * L, cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const int side = 2 * r + 1;
  for (int di = -r; di <= r; ++di)
    for (int dj = -r; dj <= r; ++dj) {
      const double fwd = resp[static_cast<int64_t>(n / 2 + di) * n + (n / 2 + dj)];
      const double bwd = resp[static_cast<int64_t>(n / 2 - di) * n + (n / 2 - dj)];
      double v = 0.5 * (fwd + bwd);
      op->stencil64[(di + r) * side + (dj + r)] = v;
      if (op->desc.euclidean && di * di + dj * dj > r * r) v = 0.0;
      op->coef.c[(di + r) * side + (dj + r)] = v;
    }
}

// Surrogate T from a reference cache file (build_surrogate's CSR, normal_ops.cpp:266-281): the
// stencil is read off the centre pixel's row, its support tells Chebyshev from Euclidean
// truncation, and every row must be exactly the clipped translation of it.
void stencil_from_tspm(tomo_op* op, const TspmFile& t) {
  check_tspm_meta(op, t, false);
  const int n = op->g.n, r = t.meta.r;
  if (r > 4 || r >= n / 2) throw ConfigError("build_surrogate: radius out of range (GPU supports 1..4)");
  const int side = 2 * r + 1;
  double st[81] = {0};
  bool present[81] = {false};
  const int64_t c = static_cast<int64_t>(n / 2) * n + n / 2;
  for (int64_t k = t.off[c]; k < t.off[c + 1]; ++k) {
    const int di = t.col[k] / n - n / 2, dj = t.col[k] % n - n / 2;
    if (di < -r || di > r || dj < -r || dj > r) throw ConfigError("TOMOSPM1: surrogate entry outside radius r");
    st[(di + r) * side + (dj + r)] = t.val[k];
    present[(di + r) * side + (dj + r)] = true;
  }
  bool euclid = false;
  for (int di = -r; di <= r; ++di)
    for (int dj = -r; dj <= r; ++dj)
      if (!present[(di + r) * side + (dj + r)]) euclid = true;
  for (int di = -r; di <= r; ++di)
    for (int dj = -r; dj <= r; ++dj)
      if (present[(di + r) * side + (dj + r)] != (!euclid || di * di + dj * dj <= r * r))
        throw ConfigError("TOMOSPM1: surrogate support is neither Chebyshev nor Euclidean");
  int64_t k = 0;
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      const int64_t row = static_cast<int64_t>(i) * n + j;
      if (t.off[row] != k) throw ConfigError("TOMOSPM1: surrogate T is not a translated stencil");
      for (int di = -r; di <= r; ++di) {
        const int ii = i + di;
        if (ii < 0 || ii >= n) continue;
        for (int dj = -r; dj <= r; ++dj) {
          const int jj = j + dj;
          if (jj < 0 || jj >= n || !present[(di + r) * side + (dj + r)]) continue;
          if (k >= t.nnz() || t.col[k] != ii * n + jj || t.val[k] != st[(di + r) * side + (dj + r)])
            throw ConfigError("TOMOSPM1: surrogate T is not a translated stencil");
          ++k;
        }
      }
    }
  if (k != t.nnz()) throw ConfigError("TOMOSPM1: surrogate T is not a translated stencil");
  op->rad = r;
  op->desc.surrogate_r = r;
  op->desc.euclidean = euclid ? 1 : 0;
  for (int q = 0; q < 81; ++q) op->stencil64[q] = q < side * side ? st[q] : 0.0;
  for (int q = 0; q < side * side; ++q) op->coef.c[q] = st[q];
}

// build_surrogate's CSR from the op's stencil (same loop order, so same bytes as save_sparse).
TspmFile surrogate_to_tspm(const tomo_op* op) {
  const int n = op->g.n, r = op->rad, side = 2 * r + 1;
  const bool euclid = op->desc.euclidean != 0;
  TspmFile t;
  t.rows = t.cols = static_cast<int64_t>(n) * n;
  t.symmetric = true;
  t.off.push_back(0);
  for (int i = 0; i < n; ++i)
    for (int j = 0; j < n; ++j) {
      for (int di = -r; di <= r; ++di) {
        const int ii = i + di;
        if (ii < 0 || ii >= n) continue;
        for (int dj = -r; dj <= r; ++dj) {
          const int jj = j + dj;
          if (jj < 0 || jj >= n) continue;
          if (euclid && di * di + dj * dj > r * r) continue;
          t.col.push_back(ii * n + jj);
          t.val.push_back(op->stencil64[(di + r) * side + (dj + r)]);
        }
      }
      t.off.push_back(static_cast<int64_t>(t.val.size()));
    }
  return t;
}

template <typename R>
double leak_probe(tomo_op* op, cudaStream_t st) {
  {
    std::lock_guard<std::mutex> lk(op->cache_mu);
    if (op->leak >= 0.0) return op->leak;
  }
  const int64_t L = op->L();
  op->ensure_batch(1);
  Scratch& S = op->W().sc;
  S.cin.ensure(L * sizeof(cplx<R>));
  S.cout.ensure(L * sizeof(cplx<R>));
  std::vector<cplx<R>> ones(L);
  for (auto& z : ones) {
    z.x = R(1);
    z.y = R(0);
  }
  CK(cudaMemcpyAsync(S.cin.p, ones.data(), sizeof(cplx<R>) * L, cudaMemcpyHostToDevice, st));
  normal_direct<R>(op, 1, S.cin.p, true, S.cout.p, st);
  launch_leak<R>(L, S.cout.as<cplx<R>>(), op->red(), st);
  SliceScalars h{};
  CK(cudaMemcpyAsync(&h, op->scal(), sizeof(SliceScalars), cudaMemcpyDeviceToHost, st));
  CK(cudaStreamSynchronize(st));
  const double leak = h.leak_den > 0.0 ? std::sqrt(h.leak_num) / std::sqrt(h.leak_den) : 0.0;
  std::lock_guard<std::mutex> lk(op->cache_mu);
  op->leak = leak;
  return leak;
}

// ---- host/device staging for the C ABI -----------------------------------------------------
const void* stage_in(const void* p, size_t bytes, Raw& buf, cudaStream_t st) {
  if (!p) return nullptr;
  if (is_device_ptr(p)) return p;
  buf.ensure(bytes);
  CK(cudaMemcpyAsync(buf.p, p, bytes, cudaMemcpyHostToDevice, st));
  return buf.p;
}

// Output either straight into a device pointer, or into `buf` and back to the host pointer.
struct OutArg {
  void* user;
  void* dev;
  size_t bytes;
  bool host;
  OutArg(void* u, size_t b, Raw& buf) : user(u), bytes(b) {
    host = !is_device_ptr(u);
    if (host) {
      buf.ensure(b);
      dev = buf.p;
    } else {
      dev = u;
    }
  }
  void finish(cudaStream_t st) {
    if (host) {
      CK(cudaMemcpyAsync(user, dev, bytes, cudaMemcpyDeviceToHost, st));
      CK(cudaStreamSynchronize(st));
    }
  }
};

// Host input and host output, several slices: stream the batch in chunks, host->device copy of
// chunk c+1 and device->host copy of chunk c-1 on their own streams while chunk c computes on
// `st` (double-buffered staging; the op's scratch is used by one chunk at a time). Pinned host
// buffers make the copies asynchronous; pageable ones still give the right answer.
template <typename F>
bool host_pipeline(tomo_op* op, int batch, const void* in, size_t in_per, void* out, size_t out_per, cudaStream_t st,
                   F&& compute) {
  if (batch < 2 || !in || !out || is_device_ptr(in) || is_device_ptr(out)) return false;
  const int chunk = std::max(1, std::min(std::max(1, op->desc.max_batch), (batch + 1) / 2));
  if (!op->W().pipe_in) {
    CK(cudaStreamCreateWithFlags(&op->W().pipe_in, cudaStreamNonBlocking));
    CK(cudaStreamCreateWithFlags(&op->W().pipe_out, cudaStreamNonBlocking));
    for (int k = 0; k < 2; ++k) {
      CK(cudaEventCreateWithFlags(&op->W().ev_in[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&op->W().ev_comp[k], cudaEventDisableTiming));
      CK(cudaEventCreateWithFlags(&op->W().ev_out[k], cudaEventDisableTiming));
    }
  }
  for (int k = 0; k < 2; ++k) {
    op->W().pin_buf[k].ensure(in_per * chunk);
    op->W().pout_buf[k].ensure(out_per * chunk);
  }
  CK(cudaEventRecord(op->W().ev_comp[0], st));  // staging free: nothing in flight yet
  CK(cudaEventRecord(op->W().ev_comp[1], st));
  CK(cudaEventRecord(op->W().ev_out[0], st));
  CK(cudaEventRecord(op->W().ev_out[1], st));
  const auto* src = static_cast<const unsigned char*>(in);
  auto* dst = static_cast<unsigned char*>(out);
  for (int c0 = 0, c = 0; c0 < batch; c0 += chunk, ++c) {
    const int nb = std::min(chunk, batch - c0), k = c & 1;
    CK(cudaStreamWaitEvent(op->W().pipe_in, op->W().ev_comp[k], 0));  // chunk c-2 no longer reads pin_buf[k]
    CK(cudaMemcpyAsync(op->W().pin_buf[k].p, src + in_per * c0, in_per * nb, cudaMemcpyHostToDevice, op->W().pipe_in));
    CK(cudaEventRecord(op->W().ev_in[k], op->W().pipe_in));
    CK(cudaStreamWaitEvent(st, op->W().ev_in[k], 0));
    CK(cudaStreamWaitEvent(st, op->W().ev_out[k], 0));  // chunk c-2 copied out of pout_buf[k]
    compute(nb, op->W().pin_buf[k].p, op->W().pout_buf[k].p);
    CK(cudaEventRecord(op->W().ev_comp[k], st));
    CK(cudaStreamWaitEvent(op->W().pipe_out, op->W().ev_comp[k], 0));
    CK(cudaMemcpyAsync(dst + out_per * c0, op->W().pout_buf[k].p, out_per * nb, cudaMemcpyDeviceToHost, op->W().pipe_out));
    CK(cudaEventRecord(op->W().ev_out[k], op->W().pipe_out));
  }
  CK(cudaStreamSynchronize(op->W().pipe_out));
  CK(cudaStreamSynchronize(st));
  return true;
}

int fail(const std::exception& e, int code) {
  g_err = e.what();
  return code;
}

template <typename F>
void with_prec(tomo_op* op, F&& f) {
  if (op->f64)
    f(double{});
  else
    f(float{});
}

}  // namespace
}  // namespace tomo_b200

#define TOMO_TRY try {
#define TOMO_CATCH                                                                   \
  return TOMO_OK;                                                                    \
  }                                                                                  \
  catch (const tomo_b200::ConfigError& e) { return fail(e, TOMO_ERR_CONFIG); }       \
  catch (const tomo_b200::NumericalError& e) { return fail(e, TOMO_ERR_NUMERICAL); } \
  catch (const tomo_b200::CudaError& e) { return fail(e, TOMO_ERR_CUDA); }           \
  catch (const tomo_b200::IoError& e) { return fail(e, TOMO_ERR_IO); }               \
  catch (const std::bad_alloc& e) { return fail(e, TOMO_ERR_CUDA); }                 \
  catch (const std::exception& e) { return fail(e, TOMO_ERR_CONFIG); }

static cudaStream_t S_(void* s) { return static_cast<cudaStream_t>(s); }

static void check_op(const tomo_op* op, int batch) {
  if (!op) throw ConfigError("null op");
  if (batch < 1) throw ConfigError("batch must be >= 1");
}

extern "C" {

const char* tomo_last_error(void) { return g_err.c_str(); }
int64_t tomo_kernel_launches(void) { return g_launches.load(); }

}  // extern "C"

namespace {
tomo_op* create_op(const tomo_geom_desc* geom, const tomo_op_desc* desc, const TspmFile* src) {
  tomo_op_desc dd{};
  if (desc) dd = *desc;
  if (dd.max_batch < 1) dd.max_batch = 1;
  if (dd.backend != TOMO_BACKEND_DIRECT && dd.backend != TOMO_BACKEND_FUSED && dd.backend != TOMO_BACKEND_SURROGATE)
    throw ConfigError("unknown backend");
  if (dd.precision != TOMO_F32 && dd.precision != TOMO_F64) throw ConfigError("unknown precision");
  int ndev = 0;
  if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0) {
    cudaGetLastError();
    throw CudaError("no CUDA device: libtomo_b200 has no CPU fallback");
  }
  if (dd.device < 0 || dd.device >= ndev) throw ConfigError("bad device ordinal");
  auto op = std::make_unique<tomo_op>();
  op->g = make_geom(geom, &dd);
  op->desc = dd;
  op->device = dd.device;
  op->f64 = dd.precision == TOMO_F64;
  op->rsz = op->f64 ? 8 : 4;
  op->src = src;
  DeviceGuard dg(op->device);
  tomo_op* o = op.get();
  Lease lease(o, nullptr);  // the build's scratch (stencil response, batch sizing)
  with_prec(o, [&](auto tag) {
    using R = decltype(tag);
    build_tables<R>(o);
    o->ensure_batch(dd.max_batch);
    if (dd.backend == TOMO_BACKEND_SURROGATE) {
      if (src)
        stencil_from_tspm(o, *src);
      else
        build_stencil<R>(o, 0);
    }
  });
  CK(cudaDeviceSynchronize());
  op->src = nullptr;
  return op.release();
}
}  // namespace

extern "C" {

int tomo_op_create(const tomo_geom_desc* geom, const tomo_op_desc* desc, tomo_op** out) {
  TOMO_TRY
  if (!out) throw ConfigError("tomo_op_create: null out");
  *out = nullptr;
  *out = create_op(geom, desc, nullptr);
  TOMO_CATCH
}

int tomo_tspm_info(const char* path, tomo_tspm_meta* info) {
  TOMO_TRY
  if (!path || !info) throw ConfigError("tomo_tspm_info: null argument");
  const TspmFile t = TspmIO::read(path, true);
  std::memset(info, 0, sizeof(*info));
  info->rows = t.rows;
  info->cols = t.cols;
  info->nnz = t.nnz();
  info->symmetric = t.symmetric ? 1 : 0;
  info->n = t.meta.n;
  info->m_sp = t.meta.m_sp;
  info->tau = t.meta.tau;
  info->angle_count = t.meta.angle_count;
  info->d = t.meta.d;
  info->r = t.meta.r;
  TOMO_CATCH
}

int tomo_op_create_tspm(const tomo_geom_desc* geom, const tomo_op_desc* desc, const char* path, tomo_op** out) {
  TOMO_TRY
  if (!out || !path) throw ConfigError("tomo_op_create_tspm: null argument");
  *out = nullptr;
  if (!desc || (desc->backend != TOMO_BACKEND_FUSED && desc->backend != TOMO_BACKEND_SURROGATE))
    throw ConfigError("tomo_op_create_tspm: backend must be fused (Gram) or surrogate (T)");
  const TspmFile t = TspmIO::read(path, true);
  *out = create_op(geom, desc, &t);
  TOMO_CATCH
}

int tomo_op_save_tspm(const tomo_op* op, const char* path, int angle_subsample_d) {
  TOMO_TRY
  if (!op || !path) throw ConfigError("tomo_op_save_tspm: null argument");
  const Geom& g = op->g;
  TspmFile t;
  if (op->desc.backend == TOMO_BACKEND_FUSED) {
    t = gram_to_tspm(op);
  } else if (op->desc.backend == TOMO_BACKEND_SURROGATE) {
    t = surrogate_to_tspm(op);
  } else {
    throw ConfigError("tomo_op_save_tspm: the direct backend has no sparse operator to save");
  }
  if (g.lo != -g.hi) throw ConfigError("TOMOSPM1: the reference format needs a symmetric window [-m_sp, m_sp]");
  if (op->sharded()) throw ConfigError("TOMOSPM1: operators are whole-geometry (not angle shards)");
  t.meta.n = g.n;
  t.meta.m_sp = g.hi;
  t.meta.tau = g.tau;
  t.meta.angle_count = g.A;
  t.meta.d = angle_subsample_d;
  t.meta.r = op->desc.backend == TOMO_BACKEND_FUSED ? 0 : op->rad;
  TspmIO::write(t, path);
  TOMO_CATCH
}

void tomo_op_destroy(tomo_op* op) {
  if (!op) return;
  DeviceGuard dg(op->device);
  delete op;
}

int tomo_op_get_info(const tomo_op* op, tomo_op_info* info) {
  TOMO_TRY
  if (!op || !info) throw ConfigError("null argument");
  std::memset(info, 0, sizeof(*info));
  info->n = op->g.n;
  info->m = op->g.m;
  info->n_b = op->g.nb;
  info->n_angles_local = op->g.a1 - op->g.a0;
  info->window = op->g.w;
  info->P = op->g.P;
  info->nnz = op->nnz;
  info->wt_rows = op->wt_rows;
  info->wt_slots = op->wt_slots;
  info->bytes_w = static_cast<int64_t>(op->Ppad) * (4 + 2 * op->g.w * static_cast<int64_t>(op->rsz));
  info->bytes_wt = op->wt_slots * (op->f64 ? 16 : 8) + static_cast<int64_t>(op->n_tasks) * 16 +
                   static_cast<int64_t>(op->g.m) * op->g.m * 2;
  info->surrogate_r = op->rad;
  info->precision = op->f64 ? TOMO_F64 : TOMO_F32;
  info->backend = op->desc.backend;
  info->gram_nnz = op->gram.nnz;
  info->gram_slots = op->gram.slots;
  info->bytes_gram = op->gram.bytes;
  info->herm_nnz = op->herm.nnz;
  info->herm_slots = op->herm.slots;
  info->herm_touched = op->herm.touched;
  info->herm_tasks = op->herm.n_tasks;
  info->sym_tasks = op->sym_ok() ? op->sym.n_tasks : 0;
  info->sym_pairs = op->sym_ok() ? op->n_paired : 0;
  info->sym_P = op->sym_ok() ? (op->sym_mode == 2 ? op->g.P : op->Ph) : 0;
  info->sym_nnz = op->sym_ok() ? op->sym.nnz : 0;
  info->sym_slots = op->sym_ok() ? op->sym.slots : 0;
  std::memcpy(info->stencil, op->stencil64, sizeof(info->stencil));
  TOMO_CATCH
}

int tomo_apply_normal(tomo_op* op, const void* in, void* out, int batch, void* stream) {
  TOMO_TRY
  check_op(op, batch);
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    if (!op->surrogate() &&
        host_pipeline(op, batch, in, op->L() * sizeof(cplx<R>), out, op->L() * sizeof(cplx<R>), st,
                      [&](int nb, const void* din, void* dout) { normal_direct<R>(op, nb, din, true, dout, st); }))
      return;
    const size_t cnt = static_cast<size_t>(batch) * op->L();
    const void* din = stage_in(in, cnt * sizeof(cplx<R>), op->W().sc.cin, st);
    OutArg o(out, cnt * sizeof(cplx<R>), op->W().sc.cout);
    if (op->surrogate()) {
      // T acts on real and imaginary parts independently (sparse.cpp:27-42)
      op->W().sc.fin.ensure(cnt * 2 * sizeof(R));
      op->W().sc.fout.ensure(cnt * 2 * sizeof(R));
      R* re = op->W().sc.fin.as<R>();
      R* im = re + cnt;
      CK(cudaMemcpy2DAsync(re, sizeof(R), din, 2 * sizeof(R), sizeof(R), cnt, cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpy2DAsync(im, sizeof(R), static_cast<const R*>(din) + 1, 2 * sizeof(R), sizeof(R), cnt,
                           cudaMemcpyDeviceToDevice, st));
      const SysParams sp = sysp(1.0, 0.0, 0.0, 0.0);
      for (int part = 0; part < 2; ++part)
        launch_stencil<R>(op->g.n, batch, op->rad, op->coef, 2, re + part * cnt, nullptr, nullptr,
                          op->W().sc.fout.as<R>() + part * cnt, nullptr, nullptr, sp, 0, op->red(), st);
      CK(cudaMemcpy2DAsync(o.dev, 2 * sizeof(R), op->W().sc.fout.p, sizeof(R), sizeof(R), cnt, cudaMemcpyDeviceToDevice,
                           st));
      CK(cudaMemcpy2DAsync(static_cast<R*>(o.dev) + 1, 2 * sizeof(R), op->W().sc.fout.as<R>() + cnt, sizeof(R), sizeof(R),
                           cnt, cudaMemcpyDeviceToDevice, st));
    } else {
      const size_t L = op->L();
      run_lanes(op, batch, st, [&](int b0, int nb, cudaStream_t ls) {
        normal_direct<R>(op, nb, static_cast<const cplx<R>*>(din) + b0 * L, true,
                         static_cast<cplx<R>*>(o.dev) + b0 * L, ls);
      });
    }
    o.finish(st);
  });
  TOMO_CATCH
}

int tomo_apply_normal_real(tomo_op* op, const void* in, void* out, int batch, void* stream) {
  TOMO_TRY
  check_op(op, batch);
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    if (!op->surrogate() &&
        host_pipeline(op, batch, in, op->L() * sizeof(R), out, op->L() * sizeof(R), st,
                      [&](int nb, const void* din, void* dout) { normal_direct<R>(op, nb, din, false, dout, st); }))
      return;
    const size_t cnt = static_cast<size_t>(batch) * op->L();
    const void* din = stage_in(in, cnt * sizeof(R), op->W().sc.fin, st);
    OutArg o(out, cnt * sizeof(R), op->W().sc.fout);
    if (op->surrogate()) {
      launch_stencil<R>(op->g.n, batch, op->rad, op->coef, 2, static_cast<const R*>(din), nullptr, nullptr,
                        static_cast<R*>(o.dev), nullptr, nullptr, sysp(1.0, 0.0, 0.0, 0.0), 0, op->red(), st);
    } else {
      const size_t L = op->L();
      run_lanes(op, batch, st, [&](int b0, int nb, cudaStream_t ls) {
        normal_direct<R>(op, nb, static_cast<const R*>(din) + b0 * L, false, static_cast<R*>(o.dev) + b0 * L, ls);
      });
    }
    o.finish(st);
  });
  TOMO_CATCH
}

int tomo_forward(tomo_op* op, const void* image, void* samples, int batch, void* stream) {
  TOMO_TRY
  check_op(op, batch);
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    const size_t cnt = static_cast<size_t>(batch) * op->L();
    const size_t scnt = static_cast<size_t>(batch) * op->g.P;
    PUpd<R> pu{};
    if (host_pipeline(op, batch, image, op->L() * sizeof(cplx<R>), samples, op->g.P * sizeof(cplx<R>), st,
                      [&](int nb, const void* din, void* dout) {
                        type2<R>(op, nb, din, true, pu, static_cast<cplx<R>*>(dout), nullptr, st);
                      }))
      return;
    const void* din = stage_in(image, cnt * sizeof(cplx<R>), op->W().sc.cin, st);
    OutArg o(samples, scnt * sizeof(cplx<R>), op->W().sc.cout);
    type2<R>(op, batch, din, true, pu, static_cast<cplx<R>*>(o.dev), nullptr, st);
    o.finish(st);
  });
  TOMO_CATCH
}

// forward_transform (fourier_slice.cpp:61-64): type-2 of a real image, through the Hermitian half grid.
int tomo_forward_real(tomo_op* op, const void* image, void* samples, int batch, void* stream) {
  TOMO_TRY
  check_op(op, batch);
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    const size_t cnt = static_cast<size_t>(batch) * op->L();
    const size_t scnt = static_cast<size_t>(batch) * op->g.P;
    PUpd<R> pu{};
    if (host_pipeline(op, batch, image, op->L() * sizeof(R), samples, op->g.P * sizeof(cplx<R>), st,
                      [&](int nb, const void* din, void* dout) {
                        type2<R>(op, nb, din, false, pu, static_cast<cplx<R>*>(dout), nullptr, st);
                      }))
      return;
    const void* din = stage_in(image, cnt * sizeof(R), op->W().sc.cin, st);
    OutArg o(samples, scnt * sizeof(cplx<R>), op->W().sc.cout);
    type2<R>(op, batch, din, false, pu, static_cast<cplx<R>*>(o.dev), nullptr, st);
    o.finish(st);
  });
  TOMO_CATCH
}

int tomo_adjoint(tomo_op* op, const void* samples, void* image, int batch, void* stream) {
  TOMO_TRY
  check_op(op, batch);
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    const size_t cnt = static_cast<size_t>(batch) * op->L();
    const size_t scnt = static_cast<size_t>(batch) * op->g.P;
    auto adj = [&](int nb, const void* din, void* dout) {
      PbEpi<R> e = plain_epi<R>(PB_COMPLEX, 1.0);
      e.out_c = static_cast<cplx<R>*>(dout);
      samples_in<R>(op, nb, static_cast<const cplx<R>*>(din), st);
      type1<R>(op, nb, e, nullptr, st);
      allreduce<R>(op, static_cast<R*>(dout), static_cast<size_t>(nb) * op->L() * 2, st);
    };
    if (host_pipeline(op, batch, samples, op->g.P * sizeof(cplx<R>), image, op->L() * sizeof(cplx<R>), st, adj))
      return;
    const void* din = stage_in(samples, scnt * sizeof(cplx<R>), op->W().sc.cin, st);
    OutArg o(image, cnt * sizeof(cplx<R>), op->W().sc.cout);
    adj(batch, din, o.dev);
    o.finish(st);
  });
  TOMO_CATCH
}

int tomo_spmv_w(tomo_op* op, const void* grid, void* samples, int batch, void* stream) {
  TOMO_TRY
  check_op(op, batch);
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    const size_t gcnt = static_cast<size_t>(batch) * op->g.m * op->g.m;
    const size_t scnt = static_cast<size_t>(batch) * op->g.P;
    const void* din = stage_in(grid, gcnt * sizeof(cplx<R>), op->W().sc.cin, st);
    OutArg o(samples, scnt * sizeof(cplx<R>), op->W().sc.cout);
    OpDev<R> d = op->dev<R>(batch);
    d.w_out_pos = 0;  // reference sample order at the API
    launch_w<R>(d, batch, static_cast<const cplx<R>*>(din), static_cast<cplx<R>*>(o.dev), nullptr, st);
    o.finish(st);
  });
  TOMO_CATCH
}

int tomo_spmv_wt(tomo_op* op, const void* samples, void* grid, int batch, void* stream) {
  TOMO_TRY
  check_op(op, batch);
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    const size_t gcnt = static_cast<size_t>(batch) * op->g.m * op->g.m;
    const size_t scnt = static_cast<size_t>(batch) * op->g.P;
    const void* din = stage_in(samples, scnt * sizeof(cplx<R>), op->W().sc.cin, st);
    OutArg o(grid, gcnt * sizeof(cplx<R>), op->W().sc.cout);
    OpDev<R> d = op->dev<R>(batch);
    launch_wt_grid<R>(d, batch, samples_in<R>(op, batch, static_cast<const cplx<R>*>(din), st),
                      static_cast<cplx<R>*>(o.dev), st);
    o.finish(st);
  });
  TOMO_CATCH
}

int tomo_backproject(tomo_op* op, double alpha, int weighted, const void* slice_data, void* out, int batch,
                     void* stream) {
  TOMO_TRY
  check_op(op, batch);
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    const size_t cnt = static_cast<size_t>(batch) * op->L();
    const size_t scnt = static_cast<size_t>(batch) * op->g.P;
    const void* din = stage_in(slice_data, scnt * sizeof(cplx<R>), op->W().sc.cin, st);
    OutArg o(out, cnt * sizeof(R), op->W().sc.fout);
    backproject<R>(op, batch, alpha, weighted != 0, static_cast<const cplx<R>*>(din), static_cast<R*>(o.dev), st);
    o.finish(st);
  });
  TOMO_CATCH
}

int tomo_cg(tomo_op* op, const tomo_system* sys, const void* rhs, const void* x0, void* x, int steps,
            double rel_tol, int batch, tomo_cg_stats* stats, void* stream) {
  TOMO_TRY
  check_op(op, batch);
  if (!sys) throw ConfigError("null system");
  if (steps < 1) throw ConfigError("cg_solve: steps must be >= 1");
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  op->ensure_batch(batch);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    const size_t cnt = static_cast<size_t>(batch) * op->L();
    Scratch& S = op->W().sc;
    const R* drhs = static_cast<const R*>(stage_in(rhs, cnt * sizeof(R), S.fin, st));
    const R* dx0 = x0 ? static_cast<const R*>(stage_in(x0, cnt * sizeof(R), S.mu1, st)) : S.zero.as<R>();
    OutArg o(x, cnt * sizeof(R), S.fout);
    CK(cudaMemsetAsync(S.sc.p, 0, sizeof(SliceScalars) * batch, st));
    cg_run<R>(op, batch, sysp(sys->alpha, sys->lambda, sys->shift, rel_tol), drhs, dx0, static_cast<R*>(o.dev),
              steps, st);
    std::vector<SliceScalars> hs(batch);
    CK(cudaMemcpyAsync(hs.data(), S.sc.p, sizeof(SliceScalars) * batch, cudaMemcpyDeviceToHost, st));
    CK(cudaStreamSynchronize(st));
    o.finish(st);
    for (int b = 0; b < batch; ++b) {
      if (hs[b].nonfinite) throw NumericalError("cg_solve diverged (non-finite iterate)");
      if (stats) {
        stats[b].steps_run = hs[b].steps_run;
        stats[b].min_ritz = std::isfinite(hs[b].min_ritz) ? hs[b].min_ritz : 0.0;
        stats[b].final_rs = hs[b].rs_last;
      }
    }
  });
  TOMO_CATCH
}

}  // extern "C"

namespace {
// split_bregman_tv (solver.cpp:219-307) for `batch` slices. Default: the whole Bregman loop is
// one CUDA graph. `record`: one graph launch for the CG and one for the Bregman update per
// iteration with CUDA events between them, giving the reference's per-iteration trace
// (t_total_s, t_cg_s; rel_l1_err against `reference` when given, update_l1).
void sb_impl(tomo_op* op, const tomo_sb_config* cfg, const void* slice_data, void* mu, int batch,
             const void* reference, double* update_l1, double* rel_l1_err, double* t_total_s, double* t_cg_s,
             tomo_sb_trace* trace, cudaStream_t st, bool record) {
  check_op(op, batch);
  if (!cfg) throw ConfigError("null config");
  if (!(cfg->alpha > 0.0)) throw ConfigError("SolverConfig: alpha must be positive");
  if (!(cfg->lambda > 0.0)) throw ConfigError("SolverConfig: lambda must be positive");
  if (cfg->max_iters < 1) throw ConfigError("SolverConfig: max_bregman_iters >= 1");
  if (cfg->cg_steps < 1) throw ConfigError("SolverConfig: cg_steps_per_update >= 1");
  if (cfg->update_tol_rel < 0.0) throw ConfigError("SolverConfig: update_tol_rel >= 0");
  if (cfg->max_iters > kMaxLoggedIters) throw ConfigError("split_bregman_tv: max_bregman_iters > 8192 not supported");
  DeviceGuard dg(op->device);
  Lease lease(op, st);
  op->ensure_batch(batch);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    const int n = op->g.n;
    const size_t cnt = static_cast<size_t>(batch) * op->L();
    const size_t scnt = static_cast<size_t>(batch) * op->g.P;
    Scratch& S = op->W().sc;
    const bool sur = op->surrogate();
    // make_subproblem (solver.cpp:164-215): sigma, then the leak probe (:236-247)
    const bool feedback = cfg->data_feedback != 0;
    double sigma = 0.0;
    if (sur)
      sigma = cfg->sigma_override >= 0.0 ? cfg->sigma_override
                                         : surrogate_sigma<R>(op, cfg->alpha, cfg->lambda, st, feedback);
    double leak = 0.0;
    if (!sur) {
      leak = leak_probe<R>(op, st);
      if (leak > 0.1) throw NumericalError("split_bregman_tv: conjugation symmetry broken");
    }
    const auto* din = static_cast<const cplx<R>*>(stage_in(slice_data, scnt * sizeof(cplx<R>), S.cin, st));
    if (feedback) {  // fk = f (solver.cpp:252), both kept in the op's internal sample order
      // sized for the op's batch capacity once, so graphs captured earlier never see them move
      const size_t fcap = static_cast<size_t>(S.cap) * op->g.P * sizeof(cplx<R>);
      if (S.fk.bytes < fcap || S.fint.bytes < fcap) {
        S.fk.ensure(fcap);
        S.fint.ensure(fcap);
        op->clear_graphs();
      }
      const cplx<R>* fi = samples_in<R>(op, batch, din, st);
      CK(cudaMemcpyAsync(S.fint.p, fi, scnt * sizeof(cplx<R>), cudaMemcpyDeviceToDevice, st));
      CK(cudaMemcpyAsync(S.fk.p, fi, scnt * sizeof(cplx<R>), cudaMemcpyDeviceToDevice, st));
    }
    backproject<R>(op, batch, cfg->alpha, sur, din, S.fid.as<R>(), st);
    // data feedback after the CG of an iteration: fk += f - F_NU^* mu_next, fid = backproject(fk)
    auto feedback_step = [&](R* mu_next, cudaStream_t cs) {
      PUpd<R> pu{};
      type2<R>(op, batch, mu_next, false, pu, nullptr, nullptr, cs);
      OpDev<R> d = op->dev<R>(batch);
      launch_feedback_samples<R>(static_cast<int64_t>(scnt), S.fk.as<cplx<R>>(), S.fint.as<cplx<R>>(), d.s, cs);
      if (sur) launch_weight_samples<R>(d.s, batch, static_cast<int>(op->g.P), op->g.nb, d.w_perm, cs);
      PbEpi<R> e = plain_epi<R>(PB_REAL, cfg->alpha);
      e.out_r = S.fid.as<R>();
      type1<R>(op, batch, e, nullptr, cs);
    };
    CK(cudaMemcpyAsync(S.rhs.p, S.fid.p, sizeof(R) * cnt, cudaMemcpyDeviceToDevice, st));
    for (auto* b : {&S.mu0, &S.bx0, &S.by0}) CK(cudaMemsetAsync(b->p, 0, sizeof(R) * cnt, st));
    std::vector<SliceScalars> init(batch);
    std::memset(init.data(), 0, sizeof(SliceScalars) * batch);
    for (auto& s : init) s.sb_tol = cfg->update_tol_rel;
    CK(cudaMemcpyAsync(S.sc.p, init.data(), sizeof(SliceScalars) * batch, cudaMemcpyHostToDevice, st));
    const SysParams sp = sysp(cfg->alpha, cfg->lambda, sigma, 0.0);
    const int iters = cfg->max_iters;
    R* mus[2] = {S.mu0.as<R>(), S.mu1.as<R>()};
    R* bxs[2] = {S.bx0.as<R>(), S.bx1.as<R>()};
    R* bys[2] = {S.by0.as<R>(), S.by1.as<R>()};
    std::vector<cudaEvent_t> ev;
    if (!record) {
      const std::string key = fmtkey("sb", batch, {cfg->alpha, cfg->lambda, sigma, double(iters), double(cfg->cg_steps),
                                                   double(cfg->warm_start), double(feedback)});
      run_graph(op, key, st, [&](cudaStream_t cs) {
        for (int it = 0; it < iters; ++it) {
          const int p = it & 1;
          cg_run<R>(op, batch, sp, S.rhs.as<R>(), cfg->warm_start ? mus[p] : S.zero.as<R>(), mus[p ^ 1],
                    cfg->cg_steps, cs);
          if (feedback) feedback_step(mus[p ^ 1], cs);
          launch_sb_post<R>(n, batch, mus[p ^ 1], mus[p], bxs[p], bys[p], bxs[p ^ 1], bys[p ^ 1], S.fid.as<R>(),
                            S.rhs.as<R>(), cfg->lambda, op->red(), cs);
          CK(cudaMemcpy2DAsync(S.upd_log.as<double>() + static_cast<size_t>(it) * batch, sizeof(double),
                               &op->scal()[0].upd, sizeof(SliceScalars), sizeof(double), batch,
                               cudaMemcpyDeviceToDevice, cs));
        }
        // final iterate lives in mus[iters & 1]; normalise its location to S.mu0
        if (iters & 1) CK(cudaMemcpyAsync(S.mu0.p, S.mu1.p, sizeof(R) * cnt, cudaMemcpyDeviceToDevice, cs));
      });
    } else {
      // the captured update graph only ever sees scratch owned by the op, sized by ensure_batch:
      // the reference is copied into S.u2 (never the caller's pointer) and rel_log holds
      // kMaxLoggedIters entries per slice, so replays after a longer solve stay in bounds
      const R* dref = nullptr;
      if (reference) {
        CK(cudaMemcpyAsync(S.u2.p, reference, cnt * sizeof(R),
                           is_device_ptr(reference) ? cudaMemcpyDeviceToDevice : cudaMemcpyHostToDevice, st));
        dref = S.u2.as<R>();
      }
      ev.resize(3 * static_cast<size_t>(iters) + 1);
      for (auto& e : ev) CK(cudaEventCreate(&e));
      CK(cudaEventRecord(ev[0], st));
      for (int it = 0; it < iters; ++it) {
        const int p = it & 1;
        run_graph(op, fmtkey("sbr_cg", batch, {cfg->alpha, cfg->lambda, sigma, double(cfg->cg_steps),
                                               double(cfg->warm_start), double(p)}),
                  st, [&](cudaStream_t cs) {
                    cg_run<R>(op, batch, sp, S.rhs.as<R>(), cfg->warm_start ? mus[p] : S.zero.as<R>(), mus[p ^ 1],
                              cfg->cg_steps, cs);
                  });
        CK(cudaEventRecord(ev[3 * it + 1], st));
        run_graph(op, fmtkey("sbr_post", batch, {cfg->lambda, double(p), dref ? 1.0 : 0.0, cfg->alpha, double(feedback)}), st, [&](cudaStream_t cs) {
          if (feedback) feedback_step(mus[p ^ 1], cs);
          launch_sb_post<R>(n, batch, mus[p ^ 1], mus[p], bxs[p], bys[p], bxs[p ^ 1], bys[p ^ 1], S.fid.as<R>(),
                            S.rhs.as<R>(), cfg->lambda, op->red(), cs);
          launch_sb_log<R>(n, batch, mus[p ^ 1], dref, S.upd_log.as<double>(),
                           dref ? S.rel_log.as<double>() : nullptr, op->red(), cs);
        });
        CK(cudaEventRecord(ev[3 * it + 2], st));
        if (it + 1 < iters) CK(cudaEventRecord(ev[3 * it + 3], st));
      }
      if (iters & 1) CK(cudaMemcpyAsync(S.mu0.p, S.mu1.p, sizeof(R) * cnt, cudaMemcpyDeviceToDevice, st));
    }
    std::vector<SliceScalars> hs(batch);
    CK(cudaMemcpyAsync(hs.data(), S.sc.p, sizeof(SliceScalars) * batch, cudaMemcpyDeviceToHost, st));
    std::vector<double> log(static_cast<size_t>(batch) * iters), rlog;
    CK(cudaMemcpyAsync(log.data(), S.upd_log.p, sizeof(double) * log.size(), cudaMemcpyDeviceToHost, st));
    if (record && reference) {
      rlog.resize(log.size());
      CK(cudaMemcpyAsync(rlog.data(), S.rel_log.p, sizeof(double) * rlog.size(), cudaMemcpyDeviceToHost, st));
    }
    CK(cudaMemcpyAsync(mu, S.mu0.p, sizeof(R) * cnt, is_device_ptr(mu) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       st));
    CK(cudaStreamSynchronize(st));
    if (record) {
      double cg_acc = 0.0;
      for (int it = 0; it < iters; ++it) {
        float t_it = 0.f, t_c = 0.f;
        CK(cudaEventElapsedTime(&t_it, ev[0], ev[3 * it + 2]));
        CK(cudaEventElapsedTime(&t_c, it == 0 ? ev[0] : ev[3 * it], ev[3 * it + 1]));
        cg_acc += t_c * 1e-3;
        if (t_total_s) t_total_s[it] = t_it * 1e-3;
        if (t_cg_s) t_cg_s[it] = cg_acc;
      }
      for (auto& e : ev) cudaEventDestroy(e);
    }
    for (int b = 0; b < batch; ++b) {
      if (hs[b].nonfinite)
        throw NumericalError(std::string("split_bregman_tv: non-finite iterate with backend ") +
                             (sur ? "surrogate" : (op->fused() ? "fused" : "direct")));
      const int ran = hs[b].sb_iters;
      for (int it = 0; it < iters; ++it) {
        const size_t o = static_cast<size_t>(b) * iters + it, l = static_cast<size_t>(it) * batch + b;
        if (update_l1) update_l1[o] = it < ran ? log[l] : 0.0;
        if (rel_l1_err && !rlog.empty()) rel_l1_err[o] = it < ran ? rlog[l] : 0.0;
      }
      if (trace) {
        trace[b].iterations = ran;
        trace[b].first_update_l1 = hs[b].first_upd;
        trace[b].sigma = sigma;
        trace[b].min_ritz = std::isfinite(hs[b].min_ritz) ? hs[b].min_ritz : 0.0;
        trace[b].imag_leakage = leak;
        trace[b].stopped_on_tolerance = hs[b].frozen;
      }
    }
  });
}
}  // namespace

extern "C" {

int tomo_split_bregman(tomo_op* op, const tomo_sb_config* cfg, const void* slice_data, void* mu, int batch,
                       double* update_l1, tomo_sb_trace* trace, void* stream) {
  TOMO_TRY
  sb_impl(op, cfg, slice_data, mu, batch, nullptr, update_l1, nullptr, nullptr, nullptr, trace, S_(stream), false);
  TOMO_CATCH
}

int tomo_split_bregman_record(tomo_op* op, const tomo_sb_config* cfg, const void* slice_data, void* mu, int batch,
                              const void* reference, double* update_l1, double* rel_l1_err, double* t_total_s,
                              double* t_cg_s, tomo_sb_trace* trace, void* stream) {
  TOMO_TRY
  sb_impl(op, cfg, slice_data, mu, batch, reference, update_l1, rel_l1_err, t_total_s, t_cg_s, trace, S_(stream),
          true);
  TOMO_CATCH
}

int tomo_tikhonov(tomo_op* op, double alpha, const void* slice_data, void* mu, int steps, double rel_tol, int batch,
                  void* stream) {
  TOMO_TRY
  check_op(op, batch);
  if (steps < 1) throw ConfigError("cg_solve: steps must be >= 1");
  if (op->surrogate()) throw ConfigError("tomo_tikhonov: direct backend only");
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  op->ensure_batch(batch);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    const size_t cnt = static_cast<size_t>(batch) * op->L();
    const size_t scnt = static_cast<size_t>(batch) * op->g.P;
    Scratch& S = op->W().sc;
    const auto* din = static_cast<const cplx<R>*>(stage_in(slice_data, scnt * sizeof(cplx<R>), S.cin, st));
    backproject<R>(op, batch, alpha, false, din, S.fid.as<R>(), st);
    CK(cudaMemsetAsync(S.sc.p, 0, sizeof(SliceScalars) * batch, st));
    const SysParams sp = sysp(alpha, 0.0, 1.0, rel_tol);
    const std::string key = fmtkey("tik", batch, {alpha, double(steps), rel_tol});
    run_graph(op, key, st,
              [&](cudaStream_t cs) { cg_run<R>(op, batch, sp, S.fid.as<R>(), S.zero.as<R>(), S.x.as<R>(), steps, cs); });
    std::vector<SliceScalars> hs(batch);
    CK(cudaMemcpyAsync(hs.data(), S.sc.p, sizeof(SliceScalars) * batch, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(mu, S.x.p, sizeof(R) * cnt, is_device_ptr(mu) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       st));
    CK(cudaStreamSynchronize(st));
    for (int b = 0; b < batch; ++b)
      if (hs[b].nonfinite) throw NumericalError("tikhonov_solve: cg diverged (non-finite iterate)");
  });
  TOMO_CATCH
}

int tomo_chambolle_pock(tomo_op* op, const tomo_cp_config* cfg, const void* slice_data, void* mu, int batch,
                        void* stream) {
  TOMO_TRY
  check_op(op, batch);
  if (!cfg || cfg->iters < 1 || cfg->cg_steps < 1) throw ConfigError("chambolle_pock: bad config");
  if (op->surrogate()) throw ConfigError("chambolle_pock: direct backend only");
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  op->ensure_batch(batch);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    const int n = op->g.n;
    const size_t cnt = static_cast<size_t>(batch) * op->L();
    const size_t scnt = static_cast<size_t>(batch) * op->g.P;
    Scratch& S = op->W().sc;
    const auto* din = static_cast<const cplx<R>*>(stage_in(slice_data, scnt * sizeof(cplx<R>), S.cin, st));
    backproject<R>(op, batch, cfg->alpha, false, din, S.fid.as<R>(), st);
    for (auto* b : {&S.mu0, &S.mu1, &S.bx0, &S.by0}) CK(cudaMemsetAsync(b->p, 0, sizeof(R) * cnt, st));
    CK(cudaMemsetAsync(S.sc.p, 0, sizeof(SliceScalars) * batch, st));
    const SysParams sp = sysp(cfg->tau_cp * cfg->alpha, 0.0, 1.0, 0.0);
    const std::string key = fmtkey("cp", batch, {cfg->alpha, cfg->lambda, cfg->tau_cp, cfg->sigma_cp, cfg->theta,
                                                 double(cfg->iters), double(cfg->cg_steps)});
    // the captured loop rotates (u^{k-1}, u^k, u^{k+1}) buffers; replay the rotation to find u^K
    R* final_u = nullptr;
    {
      R *up = S.mu1.as<R>(), *uc = S.mu0.as<R>(), *un = S.u2.as<R>();
      for (int k = 0; k < cfg->iters; ++k) {
        R* t = up;
        up = uc;
        uc = un;
        un = t;
      }
      final_u = uc;
    }
    run_graph(op, key, st, [&](cudaStream_t cs) {
      R *up = S.mu1.as<R>(), *uc = S.mu0.as<R>(), *un = S.u2.as<R>();
      R *yxo = S.bx0.as<R>(), *yxn = S.bx1.as<R>(), *yyo = S.by0.as<R>(), *yyn = S.by1.as<R>();
      for (int k = 0; k < cfg->iters; ++k) {
        launch_cp_dual<R>(n, batch, uc, up, yxo, yyo, yxn, yyn, S.fid.as<R>(), S.rhs.as<R>(), cfg->tau_cp,
                          cfg->sigma_cp, cfg->theta, cfg->lambda, cs);
        cg_run<R>(op, batch, sp, S.rhs.as<R>(), uc, un, cfg->cg_steps, cs);
        R* t = up;
        up = uc;
        uc = un;
        un = t;
        std::swap(yxo, yxn);
        std::swap(yyo, yyn);
      }
    });
    std::vector<SliceScalars> hs(batch);
    CK(cudaMemcpyAsync(hs.data(), S.sc.p, sizeof(SliceScalars) * batch, cudaMemcpyDeviceToHost, st));
    CK(cudaMemcpyAsync(mu, final_u, sizeof(R) * cnt, is_device_ptr(mu) ? cudaMemcpyDeviceToDevice : cudaMemcpyDeviceToHost,
                       st));
    CK(cudaStreamSynchronize(st));
    for (int b = 0; b < batch; ++b)
      if (hs[b].nonfinite) throw NumericalError("chambolle_pock: non-finite iterate");
  });
  TOMO_CATCH
}

int tomo_op_set_allreduce(tomo_op* op, tomo_allreduce_fn fn, void* user) {
  TOMO_TRY
  if (!op) throw ConfigError("null op");
  op->ar_fn = fn;
  op->ar_user = user;
  op->clear_all_graphs();
  TOMO_CATCH
}

int tomo_nccl_unique_id(char out[128]) {
  TOMO_TRY
  ncclUniqueId id;
  const ncclResult_t r = ncclGetUniqueId(&id);
  if (r != ncclSuccess) throw CudaError(std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
  static_assert(sizeof(id) == 128, "nccl unique id size");
  std::memcpy(out, &id, 128);
  TOMO_CATCH
}

int tomo_op_attach_nccl(tomo_op* op, const char id[128], int nranks, int rank) {
  TOMO_TRY
  if (!op) throw ConfigError("null op");
  DeviceGuard dg(op->device);
  ncclUniqueId uid;
  std::memcpy(&uid, id, 128);
  ncclComm_t comm = nullptr;
  const ncclResult_t r = ncclCommInitRank(&comm, nranks, uid, rank);
  if (r != ncclSuccess) throw CudaError(std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
  if (op->comm) ncclCommDestroy(op->comm);
  op->comm = comm;
  op->clear_all_graphs();
  TOMO_CATCH
}

int tomo_grad(int n, int precision, const void* u, void* gx, void* gy, int batch, void* stream) {
  TOMO_TRY
  if (n < 2 || batch < 1) throw ConfigError("grad: size mismatch");
  if (!is_device_ptr(u) || !is_device_ptr(gx) || !is_device_ptr(gy)) throw ConfigError("grad: device pointers required");
  if (precision == TOMO_F64)
    launch_grad<double>(n, batch, static_cast<const double*>(u), static_cast<double*>(gx), static_cast<double*>(gy),
                        S_(stream));
  else
    launch_grad<float>(n, batch, static_cast<const float*>(u), static_cast<float*>(gx), static_cast<float*>(gy),
                       S_(stream));
  TOMO_CATCH
}

int tomo_grad_adjoint(int n, int precision, const void* gx, const void* gy, void* out, int batch, void* stream) {
  TOMO_TRY
  if (n < 2 || batch < 1) throw ConfigError("grad_adjoint: size mismatch");
  if (!is_device_ptr(out) || !is_device_ptr(gx) || !is_device_ptr(gy))
    throw ConfigError("grad_adjoint: device pointers required");
  if (precision == TOMO_F64)
    launch_grad_adjoint<double>(n, batch, static_cast<const double*>(gx), static_cast<const double*>(gy),
                                static_cast<double*>(out), S_(stream));
  else
    launch_grad_adjoint<float>(n, batch, static_cast<const float*>(gx), static_cast<const float*>(gy),
                               static_cast<float*>(out), S_(stream));
  TOMO_CATCH
}

int tomo_shrink(int64_t len, int precision, const void* x, double gamma, void* out, void* stream) {
  TOMO_TRY
  if (!is_device_ptr(x) || !is_device_ptr(out)) throw ConfigError("shrink: device pointers required");
  if (precision == TOMO_F64)
    launch_shrink<double>(len, static_cast<const double*>(x), gamma, static_cast<double*>(out), S_(stream));
  else
    launch_shrink<float>(len, static_cast<const float*>(x), gamma, static_cast<float*>(out), S_(stream));
  TOMO_CATCH
}

namespace {
struct Ell {
  double intensity, a, b, cx, cy, rot;
};
void rasterize(int n, const std::vector<Ell>& es, float* img) {
  for (int i = 0; i < n; ++i) {
    const double y = -1.0 + (2.0 * i + 1.0) / n;
    for (int j = 0; j < n; ++j) {
      const double x = -1.0 + (2.0 * j + 1.0) / n;
      double v = 0.0;
      for (const auto& e : es) {
        const double c = std::cos(e.rot), s = std::sin(e.rot);
        const double dx = x - e.cx, dy = y - e.cy;
        const double u = (dx * c + dy * s) / e.a, w = (-dx * s + dy * c) / e.b;
        if (u * u + w * w <= 1.0) v += e.intensity;
      }
      img[static_cast<int64_t>(i) * n + j] = static_cast<float>(v);
    }
  }
}
}  // namespace

int tomo_shepp_logan(int n, float* img) {
  TOMO_TRY
  if (n < 4) throw ConfigError("generate_shepp_logan: n must be >= 4");
  constexpr double deg = M_PI / 180.0;
  const std::vector<Ell> t = {
      {2.00, 0.6900, 0.9200, 0.00, 0.0000, 0.0},          {-0.98, 0.6624, 0.8740, 0.00, -0.0184, 0.0},
      {-0.02, 0.1100, 0.3100, 0.22, 0.0000, -18.0 * deg}, {-0.02, 0.1600, 0.4100, -0.22, 0.0000, 18.0 * deg},
      {0.01, 0.2100, 0.2500, 0.00, 0.3500, 0.0},          {0.01, 0.0460, 0.0460, 0.00, 0.1000, 0.0},
      {0.01, 0.0460, 0.0460, 0.00, -0.1000, 0.0},         {0.01, 0.0460, 0.0230, -0.08, -0.6050, 0.0},
      {0.01, 0.0230, 0.0230, 0.00, -0.6060, 0.0},         {0.01, 0.0230, 0.0460, 0.06, -0.6050, 0.0},
  };
  rasterize(n, t, img);
  TOMO_CATCH
}

int tomo_random_ellipses(int n, int count, uint64_t seed, float* img) {
  TOMO_TRY
  if (n < 4) throw ConfigError("random_ellipses: n must be >= 4");
  std::mt19937_64 rng(seed);
  auto U = [&rng]() { return static_cast<double>(rng() >> 11) * (1.0 / 9007199254740992.0); };
  std::vector<Ell> es;
  for (int k = 0; k < count; ++k) {
    Ell e{};
    e.cx = 1.2 * U() - 0.6;
    e.cy = 1.2 * U() - 0.6;
    e.a = 0.05 + 0.35 * U();
    e.b = 0.05 + 0.35 * U();
    e.rot = M_PI * (2.0 * U() - 1.0);
    e.intensity = U();
    es.push_back(e);
  }
  rasterize(n, es, img);
  TOMO_CATCH
}

int tomo_fft_rows(int m, int rows, int precision, const void* in, void* out, int inverse, void* stream) {
  TOMO_TRY
  if (!is_device_ptr(in) || !is_device_ptr(out)) throw ConfigError("fft_rows: device pointers required");
  if (m < 32 || m > 8192 || (m & (m - 1))) throw ConfigError("fft_rows: m must be a power of two in [32, 8192]");
  // twiddle tables cached per (device, m, precision): the call is a single kernel launch
  static std::mutex mu;
  static std::map<std::tuple<int, int, int>, std::unique_ptr<Raw>> tables;
  int dev = 0;
  CK(cudaGetDevice(&dev));
  auto run = [&](auto tag) {
    using R = decltype(tag);
    const cplx<R>* twp = nullptr;
    {
      std::lock_guard<std::mutex> lk(mu);
      auto& slot = tables[std::make_tuple(dev, m, precision)];
      if (!slot) {
        std::vector<cplx<R>> tw(m);
        for (int k = 0; k < m; ++k) {
          const double ang = -2.0 * M_PI * k / m;
          tw[k].x = static_cast<R>(std::cos(ang));
          tw[k].y = static_cast<R>(std::sin(ang));
        }
        slot = std::make_unique<Raw>();
        slot->upload(tw);
      }
      twp = slot->as<cplx<R>>();
    }
    launch_fft_rows_test<R>(m, rows, twp, static_cast<const cplx<R>*>(in), static_cast<cplx<R>*>(out), inverse != 0,
                            S_(stream));
  };
  if (precision == TOMO_F64)
    run(double{});
  else
    run(float{});
  TOMO_CATCH
}

int tomo_profile_stages(tomo_op* op, int batch, int reps, int complex_io, double* ms, double* bytes, void* stream) {
  TOMO_TRY
  check_op(op, batch);
  if (!ms || !bytes || reps < 1) throw ConfigError("profile: bad arguments");
  DeviceGuard dg(op->device);
  const cudaStream_t st = S_(stream);
  Lease lease(op, st);
  op->ensure_batch(batch);
  with_prec(op, [&](auto tag) {
    using R = decltype(tag);
    const int n = op->g.n, m = op->g.m;
    const size_t cnt = static_cast<size_t>(batch) * op->L();
    Scratch& S = op->W().sc;
    // random-ish state so every kernel does its full work
    std::vector<R> h(cnt);
    std::mt19937 rng(5);
    std::normal_distribution<double> nd;
    for (auto& v : h) v = static_cast<R>(nd(rng));
    for (auto* b : {&S.r, &S.p0, &S.p1, &S.x, &S.ap, &S.mu0, &S.bx0, &S.by0, &S.fid, &S.rhs})
      CK(cudaMemcpyAsync(b->p, h.data(), sizeof(R) * cnt, cudaMemcpyHostToDevice, st));
    for (auto& v : h) v = static_cast<R>(nd(rng));  // mu_new != mu_old: the update is non-zero
    CK(cudaMemcpyAsync(S.mu1.p, h.data(), sizeof(R) * cnt, cudaMemcpyHostToDevice, st));
    std::vector<SliceScalars> init(batch);
    std::memset(init.data(), 0, sizeof(SliceScalars) * batch);
    for (auto& sc : init) {
      sc.rr[0] = sc.rr[1] = 1.0;
      sc.pap = sc.pp = 1.0;
      sc.cg_alpha = sc.cg_beta = 1e-3;
      sc.first_upd = 1e300;
    }
    const SysParams sp = sysp(1.0, 1.0, 0.0, 0.0);
    Reduce red = op->red();
    OpDev<R> d = op->dev<R>(batch);
    // the path the solvers (real images) or the complex applies (complex_io) run
    const bool herm = !complex_io && op->herm_ok() && !op->fused();
    d.herm_in = d.herm_out = herm ? 1 : 0;
    if (herm) d.Gt = d.Gth;
    const bool sym = herm && op->sym_ok();
    if (sym) op->use_sym(d);
    const size_t cbytes = sizeof(cplx<R>) * cnt;
    if (complex_io) {
      S.cin.ensure(cbytes);
      S.cout.ensure(cbytes);
      std::vector<cplx<R>> hc(cnt);
      for (auto& v : hc) v = cplx<R>{static_cast<R>(nd(rng)), static_cast<R>(nd(rng))};
      CK(cudaMemcpyAsync(S.cin.p, hc.data(), cbytes, cudaMemcpyHostToDevice, st));
      CK(cudaStreamSynchronize(st));
    }
    double acc[TOMO_NUM_STAGES] = {0};
    const bool sur = op->surrogate();
    auto launch_stage = [&](int s, cudaStream_t cs) {
      if (!sur) {
        if (s == 0 && complex_io) {
          launch_t2_rows<R>(d, batch, S.cin.p, true, PUpd<R>{}, cs);
        } else if (s == 0) {
          PUpd<R> pu{};
          pu.enabled = 1;
          pu.r = S.r.as<R>();
          pu.p = S.p0.as<R>();
          pu.step = 1;
          pu.red = red;
          if (cgcg_on() && !op->sharded()) {  // the fused C-G update (both recurrences live)
            pu.cgcg = 1;
            pu.step = 2;
            pu.s = S.p1.as<R>();
            pu.w = S.ap.as<R>();
            pu.x = S.x.as<R>();
          }
          launch_t2_rows<R>(d, batch, S.p0.p, false, pu, cs);
        } else if (s == 1) {
          launch_t2_cols<R>(d, batch, op->scal(), cs);
        } else if (s == 2) {
          if (op->fused())
            launch_gram<R>(d, batch, d.g, d.Gt, op->scal(), cs);
          else {
            if (d.s_stride == 2 * d.P && op->n_units > 0) {
              launch_w_pair<R>(d, op->pair_w<R>(), batch, d.g, d.s, op->scal(), cs);
            } else {
              launch_w<R>(d, batch, d.g, d.s, op->scal(), cs);
              if (d.s_stride == 2 * d.P)
                launch_pair_sigma<R>(d.s, batch, d.P, d.s_stride, op->ppos.as<int>(), cs);
            }
          }
        } else if (s == 3) {
          if (!op->fused()) launch_wt_spread<R>(d, batch, d.s, d.Gt, op->scal(), cs);
        } else if (s == 4) {
          launch_t1_cols_only<R>(d, batch, op->scal(), cs);
        } else if (s == 5 && complex_io) {
          PbEpi<R> e = plain_epi<R>(PB_COMPLEX, 1.0);
          e.out_c = S.cout.as<cplx<R>>();
          launch_t1_rows<R>(d, batch, e, cs);
        } else if (s == 5) {
          PbEpi<R> e = plain_epi<R>(PB_CG_STEP, 1.0);
          e.p = S.p0.as<R>();
          e.ap = S.ap.as<R>();
          e.sys = sp;
          e.step = 1;
          e.red = red;
          launch_t1_rows<R>(d, batch, e, cs);
        }
      } else if (s == 8) {
        launch_stencil<R>(n, batch, op->rad, op->coef, 0, S.p0.as<R>(), S.r.as<R>(), S.p1.as<R>(), S.ap.as<R>(),
                          nullptr, nullptr, sp, 1, red, cs);
      }
      if (s == 6) {
        if (!sur && cgcg_on() && !op->sharded())  // C-G: one final update per CG call
          launch_cgcg_final<R>(n, batch, S.ap.as<R>(), S.p0.as<R>(), S.p1.as<R>(), S.x.as<R>(), S.r.as<R>(), sp, 2,
                               red, cs);
        else
          launch_cg_update<R>(n, batch, S.p0.as<R>(), S.ap.as<R>(), S.x.as<R>(), S.r.as<R>(), sp, 1, red, cs);
      }
      if (s == 7)
        launch_sb_post<R>(n, batch, S.mu1.as<R>(), S.mu0.as<R>(), S.bx0.as<R>(), S.by0.as<R>(), S.bx1.as<R>(),
                          S.by1.as<R>(), S.fid.as<R>(), S.rhs.as<R>(), 1.0, red, cs);
    };
    CK(cudaMemcpyAsync(S.sc.p, init.data(), sizeof(SliceScalars) * batch, cudaMemcpyHostToDevice, st));
    cudaEvent_t e0, e1;
    CK(cudaEventCreate(&e0));
    CK(cudaEventCreate(&e1));
    auto stage_on = [&](int s) {
      return sur ? (s >= 6) : (s <= 7 && !(op->fused() && s == 3));
    };
    for (int s = 0; s < TOMO_NUM_STAGES; ++s) {
      const bool on = stage_on(s);
      if (!on) continue;
      // each stage timed as a CUDA graph of `reps` back-to-back launches (no host launch gaps)
      const std::string key = fmtkey("prof", batch, {double(s), double(reps)});
      CK(cudaMemcpyAsync(S.sc.p, init.data(), sizeof(SliceScalars) * batch, cudaMemcpyHostToDevice, st));
      run_graph(op, key, st, [&](cudaStream_t cs) {
        for (int r = 0; r < reps; ++r) launch_stage(s, cs);
      });  // warm-up launch + instantiation
      CK(cudaMemcpyAsync(S.sc.p, init.data(), sizeof(SliceScalars) * batch, cudaMemcpyHostToDevice, st));
      CK(cudaEventRecord(e0, st));
      run_graph(op, key, st, [&](cudaStream_t) {});
      CK(cudaEventRecord(e1, st));
      CK(cudaEventSynchronize(e1));
      float t = 0.f;
      CK(cudaEventElapsedTime(&t, e0, e1));
      acc[s] = t;
    }
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    const double B = batch, nn = static_cast<double>(n) * n, mn = static_cast<double>(m) * n,
                 mm = static_cast<double>(m) * m, P = static_cast<double>(op->g.P), rs = sizeof(R), cs = 2 * sizeof(R);
    double by[TOMO_NUM_STAGES] = {0};
    if (!sur) {
      // Hermitian half grid: m/2 + 1 of the m grid rows (H, g, spread grid, K)
      const double rows = herm ? m / 2 + 1 : m, hn = rows * n, hm = rows * m;
      const double in0 = complex_io ? cs * nn : cgcg_on() && !op->sharded()
                                                     ? 9 * rs * nn   // C-G: read r, w, x, p, s; write p, s, x, r
                                                     : 3 * rs * nn;  // read p, r; write p
      by[0] = B * (in0 + cs * hn);                         // + write H
      by[1] = B * (cs * hn + cs * hm);                     // read H, write g
      // SURVEY.md §8(d) algorithmic bytes (payload only, no implementation padding):
      //   W:   (4 + r) nnz + c T + c P         (ELL entries, gather of the T touched nodes, samples)
      //   W^T: (4 + r) nnz + 8 (T + 1) + c P + c G  (entries, row pointers + ids, samples, grid)
      // the matrix stream is read once per launch, the vectors once per slice
      //   (the Hermitian path: W gathers the T_h touched nodes of the half grid; the folded W^T
      //    streams its nnz_f entries, ids of T_h nodes, writes the half grid)
      //   (mirror pairs: W runs on the Ph kept samples, the primaries' fold streams its entries)
      //   (overlap pairs: W evaluates every sample and the pair sums)
      const bool half_w = sym && op->sym_mode == 1;
      const double Pw = half_w ? static_cast<double>(op->Ph) : P;
      const double nnzb = (half_w ? Pw * op->g.w * op->g.w : static_cast<double>(op->nnz)) * (4.0 + rs);
      // (pair sums: one write per pair from the unit W, or the pass: two reads and a write per pair)
      const double sig = sym && op->sym_mode == 2
                             ? B * (op->n_units > 0 ? 0.5 : 1.5) * cs * static_cast<double>(op->n_paired) / 2.0
                             : 0.0;
      const double T = static_cast<double>(herm ? op->herm.touched : op->wt_rows);
      const double nnzt = sym ? static_cast<double>(op->sym.nnz) * (4.0 + rs)
                              : herm ? static_cast<double>(op->herm.nnz) * (4.0 + rs) : nnzb;
      by[2] = op->fused()  // Gram stream, read + write touched nodes
                  ? static_cast<double>(op->gram.bytes) + B * (2 * cs * op->wt_rows)
                  : nnzb + B * (cs * T + cs * Pw) + sig;
      by[3] = nnzt + 8.0 * (T + 1) + B * (cs * (Pw + (sig > 0 ? op->n_paired / 2.0 : 0.0)) + cs * hm);
      by[4] = B * (cs * hm + cs * hn);                     // read spread grid, write K
      by[5] = B * (cs * hn + (complex_io ? cs * nn : 2 * rs * nn));  // read K (+ p); write Ap / out
    } else {
      by[8] = B * 4 * rs * nn;  // read r, p; write p, Ap
    }
    by[6] = B * (!sur && cgcg_on() && !op->sharded() ? 7 : 6) * rs * nn;  // read x, r, p, Ap (C-G: + s); write x, r
    by[7] = B * 8 * rs * nn;  // read mu_new, mu_old, bx, by, fid; write bx, by, rhs
    for (int k = 0; k < TOMO_NUM_STAGES; ++k) {
      const bool on = stage_on(k);
      ms[k] = on ? acc[k] / reps : 0.0;
      bytes[k] = on ? by[k] : 0.0;
    }
  });
  TOMO_CATCH
}

}  // extern "C"
