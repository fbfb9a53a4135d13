// se2map.cu — C-ABI runtime of libse2map.so (see include/se2map.h for the contract).
//
// Owns the device state of one robot-centric map: the ring-buffered elevation window
// (Eq. 4), the per-yaw footprint tables (reading R5), the output planes,
// the dirty-region tracker for INCREMENTAL assessment, and the TMA descriptor of the map.
#include <math.h>
#include <stdio.h>
#include <string.h>

#include <algorithm>
#include <new>
#include <string>
#include <vector>

#include "../../include/se2map.h"
#include "nccl_dl.h"
#include "se2m_internal.h"

#ifndef SE2M_PERIOD
#define SE2M_PERIOD 36       // yaw-chain restart period on large maps (A/B knob; 9 / 12 / 18 measured slower)
#endif
#ifndef SE2M_TSPLIT
#define SE2M_TSPLIT 1        // vertical-window-edge tiles in their own concurrent kernel (A/B knob)
#endif

using namespace se2m;

namespace {

struct Rect {  // world cells [I0, I1) x [J0, J1)
  long long I0, I1, J0, J1;
};

long long floor_div(long long a, long long b) {
  long long q = a / b;
  if ((a % b != 0) && ((a < 0) != (b < 0))) --q;
  return q;
}
int pmod(long long a, int n) {
  long long m = a % n;
  return (int)(m < 0 ? m + n : m);
}

std::string g_init_error;  // message of the last failed se2m_init

}  // namespace

struct se2m_map {
  se2m_params prm;
  cudaStream_t stream = nullptr;
  bool own_stream = false;
  int H = 0, paired = 0, R = 0, R_T = 0, ldh = 0, trav_words = 0;
  int k_lo = 0, k_hi = 0;  // owned representative bins [k_lo, k_hi)
  long long I_M = 0, J_M = 0;
  float* d_h = nullptr;
  float4* d_out = nullptr;  // state records [k][ny][nx] (risk, pitch, roll, z), ring layout
  uint32_t* d_trav = nullptr;
  float* d_sdf = nullptr;    // NEXT-2: SDF layers (representative bins), ring layout
  uint16_t* d_sdf_g = nullptr;  // NEXT-2 scratch: column distances
  float* d_var = nullptr;    // NEXT-1: cell height variance, ring layout like d_h
  FrontendScratch fe{};
  float* d_pts = nullptr;
  size_t pts_cap = 0;
  bool sdf_valid = false;
  double sdf_dmax = 0;
  int4* d_full = nullptr;   // run-entry tables (see AssessParams)
  int4* d_full_fmt = nullptr;
  int* d_segb = nullptr;              // [seg + 1] yaw-chain segment bounds
  unsigned char* d_seg_rst = nullptr; // [H] chain restart flags
  // the vertical-window-edge kernel's own yaw chain (seg_e >= seg segments: its CTAs take fewer bins, so that
  // they stop being the critical path of small launches, e.g. the row bands of 8 ranks); aliases the main
  // tables when seg_e == seg
  int seg_e = 1;
  std::vector<int> chain_off_e, chain_mid_e;
  int4* d_chain_e = nullptr;
  int* d_chain_off_e = nullptr;
  int* d_chain_mid_e = nullptr;
  int* d_segb_e = nullptr;
  unsigned char* d_seg_rst_e = nullptr;
  bool own_edge_tables = false;
  int* d_full_off = nullptr;
  int4* d_chain = nullptr;
  int* d_chain_off = nullptr;
  std::vector<int> full_off, chain_off, chain_mid;
  int* d_chain_mid = nullptr;
  int seg = 1;  // yaw-chain segments (AssessParams::seg; H = no chain)
  float4* d_geo = nullptr;
  float4* d_geoc = nullptr;
  float2* d_cs = nullptr;
  std::vector<int> ncells;  // |P_k| per rep bin
  float* d_stage = nullptr;  // update / download staging
  size_t stage_bytes = 0;
  double* d_qxyt = nullptr;   // query staging: xyt in, 5 x n floats out, out-of-range counter
  float* d_qout = nullptr;
  int* d_qcnt = nullptr;
  size_t q_cap = 0;
  CUtensorMap tmap;
  bool tma_ok = false;
  int smem_optin = 227 * 1024;  // cudaDevAttrMaxSharedMemoryPerBlockOptin of the device
  int n_sm = 148;               // cudaDevAttrMultiProcessorCount of the device
  int slots_per_sm = 0;         // resident assess CTAs per SM (occupancy API, first assess)
  // NEXT-4: nearest-neighbour inpainted view (ring layout like d_h), allocated on first use
  float* d_hin = nullptr;
  int* d_site = nullptr;
  int* d_ipc = nullptr;      // [0] known cells, [1..4] changed-cell box (logical i0, i1, j0, j1)
  int* h_ipc = nullptr;      // pinned copy
  CUtensorMap tmap_in;
  bool tma_in_ok = false;
  bool inpaint_valid = false;
  // se2m_download_compact_rep: copy stream, double-buffered staging, events (created on first use)
  cudaStream_t copy_stream = nullptr;
  // assess: the vertical-window-edge tiles' kernel runs on this stream, forked from / joined into `stream`
  cudaStream_t edge_stream = nullptr;
  cudaEvent_t ev_fork = nullptr, ev_join = nullptr;
  cudaEvent_t ev_gathered[2] = {nullptr, nullptr}, ev_copied[2] = {nullptr, nullptr};
  char* d_rep[2] = {nullptr, nullptr};
  size_t rep_bytes = 0;
  int rep_slot = 0;
  bool force_general = false;  // a full stencil is degenerate (R22): every tile takes the general path
  bool have_data = false;
  bool all_dirty = true;
  std::vector<Rect> dirty;
  long long launches = 0;
  // row-band halo transport (se2m_exchange_halo): the library's NCCL communicator and its 4 device slab
  // buffers (to g - 1, to g + 1, from g + 1, from g - 1), allocated on first use
  ncclComm_t comm = nullptr;
  // se2m_step as a CUDA graph (params.step_graph): the executable graph, updated in place every step
  cudaGraphExec_t step_exec = nullptr;
  bool step_warm = false;  // one direct step ran (lazy allocations / attributes done before any capture)
  float* d_halo[4] = {nullptr, nullptr, nullptr, nullptr};
  std::string err;
};

// ------------------------------------------------------------------------------------------
static se2m_status fail(se2m_map* m, se2m_status st, const std::string& msg) {
  if (m) m->err = msg;
  else g_init_error = msg;
  return st;
}
static se2m_status cuda_fail(se2m_map* m, cudaError_t e, const char* what) {
  return fail(m, SE2M_ERR_CUDA, std::string(what) + ": " + cudaGetErrorString(e));
}
// Every handle call runs on the handle's device and restores the caller's current device on return
// (two maps on two GPUs in one thread must not see each other's device selection).
struct DevGuard {
  int prev = -1;
  explicit DevGuard(int dev) {
    int cur = -1;
    if (cudaGetDevice(&cur) == cudaSuccess && cur != dev && cudaSetDevice(dev) == cudaSuccess) prev = cur;
  }
  ~DevGuard() {
    if (prev >= 0) cudaSetDevice(prev);
  }
  DevGuard(const DevGuard&) = delete;
  DevGuard& operator=(const DevGuard&) = delete;
};
#define SE2M_ENTER(m)                          \
  if (!(m)) return SE2M_ERR_INVALID_ARG;       \
  DevGuard dev_guard_((m)->prm.device)
#define CUDA_TRY(m, call, what)                         \
  do {                                                  \
    cudaError_t e_ = (call);                            \
    if (e_ != cudaSuccess) return cuda_fail(m, e_, what); \
  } while (0)

static int pick_radius(int R) {
  for (int r : kRadii)
    if (r >= R) return r;
  return -1;
}

// Footprint stencil, reading R5 (rule C5 of SURVEY.md §8(c)): cell centres, q in cell units with the
// representative angle theta_k (k < H), include iff q <= 1 + 1e-9.  FP64 on the host, once.
static bool build_stencils(se2m_map* m, std::vector<int4>& runs, std::vector<int>& nrows, std::vector<float4>& geo, std::vector<float4>& geoc,
                           std::vector<float2>& cs) {
  const se2m_params& P = m->prm;
  const double a = P.ellipse_ex / P.resolution, b = P.ellipse_ey / P.resolution;
  const int Rs = (int)ceil(std::max(a, b)) + 1;
  struct Run { int lo, hi; };
  std::vector<std::vector<Run>> rr(m->H, std::vector<Run>(2 * Rs + 1, Run{0, -1}));
  int R = 0;
  m->ncells.assign(m->H, 0);
  std::vector<long long> Sxx(m->H, 0), Sxy(m->H, 0), Syy(m->H, 0);
  cs.resize(m->H);
  for (int k = 0; k < m->H; ++k) {
    const double th = -M_PI + 2.0 * M_PI * (double)k / (double)P.n_yaw;
    const double c = cos(th), s = sin(th);
    cs[k] = make_float2((float)c, (float)s);
    for (int dj = -Rs; dj <= Rs; ++dj) {
      int lo = 1 << 30, hi = -(1 << 30), cnt = 0;
      for (int di = -Rs; di <= Rs; ++di) {
        const double u = di * c + dj * s, v = -di * s + dj * c;
        const double q = (u / a) * (u / a) + (v / b) * (v / b);
        if (q <= 1.0 + 1e-9) {
          lo = std::min(lo, di); hi = std::max(hi, di); ++cnt;
          m->ncells[k]++;
          Sxx[k] += (long long)di * di; Sxy[k] += (long long)di * dj; Syy[k] += (long long)dj * dj;
          R = std::max(R, std::max(std::abs(di), std::abs(dj)));
        }
      }
      if (cnt) {
        if (cnt != hi - lo + 1) return false;  // an ellipse row must be one run (convexity)
        rr[k][dj + Rs] = Run{lo, hi};
      }
    }
  }
  m->R = R;
  m->R_T = pick_radius(std::max(R, 1));
  if (m->R_T < 0) return false;
  const int NR = 2 * m->R_T + 1;
  runs.assign((size_t)m->H * NR, make_int4(0, -1, 0, 0));
  nrows.assign(m->H, 0);
  geo.resize(m->H);
  geoc.resize(4 * (size_t)m->H);
  for (int k = 0; k < m->H; ++k) {
    // full-stencil covariance of the cell-centre offsets, metres^2, FP64 then rounded (Sx = Sy = 0)
    const double N = m->ncells[k], r = P.resolution;
    const double c00 = r * r * Sxx[k] / N, c01 = r * r * Sxy[k] / N, c11 = r * r * Syy[k] / N;
    // eigen-decomposition of the footprint geometry A = [[c00, c01], [c01, c11]] = a1 q1 q1^T + a2 q2 q2^T
    // (a1 <= a2, q2 = (-q1y, q1x)), and the projections of q1, q2 on the bin's heading e = (cos, sin) and
    // on (sin, -cos): the interior-tile solver works in this basis (assess.cu, arrow2)
    const double hm = 0.5 * (c00 + c11), hd = 0.5 * (c00 - c11);
    const double rad = sqrt(hd * hd + c01 * c01);
    const double a1 = hm - rad, a2 = hm + rad;
    const double psi = 0.5 * atan2(2.0 * c01, c00 - c11);  // direction of the a2 axis
    const double q1x = -sin(psi), q1y = cos(psi), q2x = -q1y, q2y = q1x;
    const double th = -M_PI + 2.0 * M_PI * (double)k / (double)P.n_yaw, ct = cos(th), st = sin(th);
    geoc[4 * k] = make_float4((float)c00, (float)c01, (float)c11, (float)(1.0 / N));
    geoc[4 * k + 1] = make_float4((float)(r / N), (float)a1, (float)a2, (float)(a1 + a2));
    geoc[4 * k + 2] = make_float4((float)q1x, (float)q1y, (float)(q1x * ct + q1y * st), (float)(q2x * ct + q2y * st));
    geoc[4 * k + 3] = make_float4((float)(q1x * st - q1y * ct), (float)(q2x * st - q2y * ct), 0.f, 0.f);
    for (int dj = -std::min(Rs, m->R_T); dj <= std::min(Rs, m->R_T); ++dj) {
      const Run& q = rr[k][dj + Rs];
      if (q.hi >= q.lo) runs[(size_t)k * NR + nrows[k]++] = make_int4(q.lo, q.hi, dj + m->R_T, 0);
    }
    geo[k] = make_float4((float)m->ncells[k], (float)Sxx[k], (float)Sxy[k], (float)Syy[k]);
    const double det2 = (double)Sxx[k] * Syy[k] - (double)Sxy[k] * Sxy[k];  // Sx = Sy = 0 (point symmetry)
    if (m->ncells[k] < 3 || !(det2 > 0)) m->force_general = true;
  }
  return true;
}

// Run-entry tables (AssessParams::full / chain) from the per-bin row runs: element offsets into a
// halo prefix row of pitch PW = TX + 2 R_T + 1, relative to the state's own column.
#ifndef SE2M_CELL_MAX
#define SE2M_CELL_MAX 2  // endpoint moves of up to this many cells become single-cell chain entries
#endif

// Full rows of every bin (border tiles, the direct path): run entries (e-, e+, d, 0) -> m->full_off.
static void build_full(se2m_map* m, const std::vector<int4>& runs, const std::vector<int>& nrows,
                       std::vector<int4>& full) {
  const int RT = m->R_T, NR = 2 * RT + 1, PW = TX + 2 * RT + 1;
  m->full_off.assign(m->H + 1, 0);
  full.clear();
  for (int k = 0; k < m->H; ++k) {
    m->full_off[k] = (int)full.size();
    for (int i = 0; i < nrows[k]; ++i) {
      const int4 q = runs[(size_t)k * NR + i];  // (lo, hi, d)
      full.push_back(make_int4(q.z * PW + RT + q.x, q.z * PW + RT + q.y + 1, q.z, 0));
    }
  }
  m->full_off[m->H] = (int)full.size();
}

// The yaw-chain table for S segments (restarts at the bounds floor(H s / S)), in the kernel's shared-memory
// format: per bin the prefix entries, then (from chain_mid[k]) the single-cell entries.
static void build_chain(const se2m_map* m, const std::vector<int4>& runs, const std::vector<int>& nrows, int S,
                        std::vector<int4>& chain, std::vector<int>& chain_off, std::vector<int>& chain_mid) {
  const int RT = m->R_T, NR = 2 * RT + 1, PW = TX + 2 * RT + 1;
  auto row_runs = [&](int k) {  // d -> (a, b) or (0, -1)
    std::vector<int2> r(NR, make_int2(0, -1));
    for (int i = 0; i < nrows[k]; ++i) {
      const int4 q = runs[(size_t)k * NR + i];
      r[q.z] = make_int2(q.x, q.y);
    }
    return r;
  };
  auto ea = [&](int d, int a) { return d * PW + RT + a; };
  auto eb = [&](int d, int b) { return d * PW + RT + b + 1; };
  auto fbits = [](float f) { int i; memcpy(&i, &f, 4); return i; };
  // chain prefix entry in shared-memory format: run sum = P[y] - P[x] (byte offsets into {P0,P2} / PX)
  auto pent = [&](int x, int y, int d) { return make_int4(8 * x, 8 * y, 4 * x, fbits((float)(d - RT))); };
  auto cent = [&](int d, int di, int sg) {
    return make_int4(4 * ea(d, di), fbits((float)sg), fbits((float)(sg * di)), fbits((float)(sg * (d - RT))));
  };
  chain_off.assign(m->H + 1, 0);
  chain_mid.assign(m->H, 0);
  chain.clear();
  std::vector<int2> prev;
  for (int k = 0; k < m->H; ++k) {
    const std::vector<int2> cur = row_runs(k);
    chain_off[k] = (int)chain.size();
    std::vector<int4> cells;
    if (seg_restart(m->H, S, k)) {
      for (int d = 0; d < NR; ++d)
        if (cur[d].y >= cur[d].x) chain.push_back(pent(ea(d, cur[d].x), eb(d, cur[d].y), d));
    } else {
      // run(k) - run(k-1) per row: cells [lo, hi] entering (sg = +1) or leaving (-1); <= 2 cells become
      // cell entries, longer spans a prefix entry P[eb(hi)] - P[ea(lo)] (sign by endpoint order)
      auto span = [&](int d, int lo, int hi, int sg) {
        if (hi < lo) return;
        if (hi - lo + 1 <= SE2M_CELL_MAX) {
          for (int di = lo; di <= hi; ++di) cells.push_back(cent(d, di, sg));
        } else if (sg > 0) {
          chain.push_back(pent(ea(d, lo), eb(d, hi), d));
        } else {
          chain.push_back(pent(eb(d, hi), ea(d, lo), d));
        }
      };
      for (int d = 0; d < NR; ++d) {
        const bool e1 = prev[d].y < prev[d].x, e2 = cur[d].y < cur[d].x;
        if (e1 && e2) continue;
        if (e1) { span(d, cur[d].x, cur[d].y, +1); continue; }
        if (e2) { span(d, prev[d].x, prev[d].y, -1); continue; }
        if (cur[d].x < prev[d].x) span(d, cur[d].x, prev[d].x - 1, +1);
        if (cur[d].x > prev[d].x) span(d, prev[d].x, cur[d].x - 1, -1);
        if (cur[d].y > prev[d].y) span(d, prev[d].y + 1, cur[d].y, +1);
        if (cur[d].y < prev[d].y) span(d, cur[d].y + 1, prev[d].y, -1);
      }
    }
    chain_mid[k] = (int)chain.size();
    chain.insert(chain.end(), cells.begin(), cells.end());
    prev = cur;
  }
  chain_off[m->H] = (int)chain.size();
}

static void build_tables(se2m_map* m, const std::vector<int4>& runs, const std::vector<int>& nrows,
                         std::vector<int4>& full, std::vector<int4>& chain) {
  build_full(m, runs, nrows, full);
  build_chain(m, runs, nrows, m->seg, chain, m->chain_off, m->chain_mid);
}

static bool make_tensor_map(se2m_map* m, CUtensorMap* tm, float* base) {
  typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                               const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                               CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult qres;
  if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &qres) != cudaSuccess || !fn ||
      qres != cudaDriverEntryPointSuccess)
    return false;
  const int HX = TX + 2 * m->R_T, HY = tile_rows(m->R_T) + 2 * m->R_T;
  if (HX > 256 || HY > 256 || HX > m->prm.nx || HY > m->prm.ny) return false;
  cuuint64_t dims[2] = {(cuuint64_t)m->prm.nx, (cuuint64_t)m->prm.ny};
  cuuint64_t strides[1] = {(cuuint64_t)m->ldh * 4};
  cuuint32_t box[2] = {(cuuint32_t)HX, (cuuint32_t)HY};
  cuuint32_t estr[2] = {1, 1};
  CUresult r = ((EncodeFn)fn)(tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2, base, dims, strides, box, estr,
                              CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                              CU_TENSOR_MAP_L2_PROMOTION_L2_128B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  return r == CUDA_SUCCESS;
}

static AssessParams make_params(const se2m_map* m) {
  AssessParams p;
  memset(&p, 0, sizeof p);
  p.nx = m->prm.nx; p.ny = m->prm.ny; p.ldh = m->ldh;
  p.I_M = m->I_M; p.J_M = m->J_M;
  p.h = m->d_h;
  p.pxM = pmod(m->I_M, m->prm.nx); p.pyM = pmod(m->J_M, m->prm.ny);
  p.out = m->d_out; p.trav = m->d_trav;
  p.trav_words = m->trav_words;
  p.n_yaw = m->prm.n_yaw; p.H = m->H; p.paired = m->paired; p.R = m->R;
  p.full = m->d_full; p.full_fmt = m->d_full_fmt; p.full_off = m->d_full_off; p.chain = m->d_chain; p.chain_off = m->d_chain_off; p.chain_mid = m->d_chain_mid;
  p.seg = m->seg; p.seg_chunk = 1; p.n_chunks = 0;
  p.segb = m->d_segb; p.seg_rst = m->d_seg_rst;
  p.geo = m->d_geo; p.geoc = m->d_geoc; p.cs = m->d_cs;
  p.r = (float)m->prm.resolution;
  p.kappa_max = (float)m->prm.kappa_max; p.phi_x_max = (float)m->prm.phi_x_max; p.phi_y_max = (float)m->prm.phi_y_max;
  p.wk = (float)(m->prm.w_r[0] / m->prm.kappa_max);
  p.wx = (float)(m->prm.w_r[1] / m->prm.phi_x_max);
  p.wy = (float)(m->prm.w_r[2] / m->prm.phi_y_max);
  // the launch starts at the chain restart at or before the first owned bin (replayed, not stored)
  p.seg_first = seg_of(m->H, m->seg, m->k_lo);
  p.k_begin = seg_bound(m->H, m->seg, p.seg_first); p.k_end = m->k_hi; p.k_store = m->k_lo;
  p.k_chunk = 1;
  p.use_tma = m->tma_ok ? 1 : 0;
  p.force_general = m->force_general ? 1 : 0;
  const bool rows = m->prm.shard_mode == SE2M_SHARD_ROWS && m->prm.world_size > 1;
  p.own_G = rows ? m->prm.world_size : 1;
  p.own_rank = rows ? m->prm.rank : 0;
  p.own_ty = tile_rows(m->R_T);
  return p;
}

static se2m_status ensure_stage(se2m_map* m, size_t bytes) {
  if (m->stage_bytes >= bytes) return SE2M_OK;
  if (m->d_stage) { cudaStreamSynchronize(m->stream); cudaFree(m->d_stage); m->d_stage = nullptr; m->stage_bytes = 0; }
  CUDA_TRY(m, cudaMalloc(&m->d_stage, bytes), "cudaMalloc(staging)");
  m->stage_bytes = bytes;
  return SE2M_OK;
}

// ------------------------------------------------------------------------------------------
extern "C" void se2m_default_params(se2m_params* p) {
  if (!p) return;
  memset(p, 0, sizeof *p);
  p->nx = 100; p->ny = 100; p->n_yaw = 36;
  p->resolution = 0.1;
  p->ellipse_ex = 0.8; p->ellipse_ey = 0.5;
  p->w_r[0] = 0.4; p->w_r[1] = 0.3; p->w_r[2] = 0.3;
  p->kappa_max = 0.1; p->phi_x_max = 0.52; p->phi_y_max = 0.52;
  p->world_size = 1;
  p->fe_z_min = -1.5; p->fe_z_max = 1.5; p->fe_gate = 2.0; p->fe_ray_eps = 0.05; p->fe_prior_var = 1e-4;
  p->step_graph = 0;  // (measured: no gain on the stream step, whose device time is the assess kernel's)
}

static se2m_status validate(const se2m_params* p) {
  if (!p) return fail(nullptr, SE2M_ERR_INVALID_ARG, "params is NULL");
  if (p->nx < 1 || p->ny < 1 || (long long)p->nx * p->ny > (1ll << 31)) return fail(nullptr, SE2M_ERR_INVALID_ARG, "nx, ny must be >= 1 and nx*ny <= 2^31");
  if (p->n_yaw < 1 || p->n_yaw > 4096) return fail(nullptr, SE2M_ERR_INVALID_ARG, "n_yaw must be in [1, 4096]");
  if (!(p->resolution > 0) || !isfinite(p->resolution)) return fail(nullptr, SE2M_ERR_INVALID_ARG, "resolution must be > 0");
  if (!(p->ellipse_ex > 0) || !(p->ellipse_ey > 0)) return fail(nullptr, SE2M_ERR_INVALID_ARG, "ellipse semi-axes must be > 0");
  for (int i = 0; i < 3; ++i)
    if (!(p->w_r[i] >= 0)) return fail(nullptr, SE2M_ERR_INVALID_ARG, "w_r must be >= 0");
  if (!(p->kappa_max > 0) || !(p->phi_x_max > 0) || !(p->phi_y_max > 0)) return fail(nullptr, SE2M_ERR_INVALID_ARG, "limits must be > 0");
  if (!isfinite(p->robot_x) || !isfinite(p->robot_y)) return fail(nullptr, SE2M_ERR_INVALID_ARG, "robot position must be finite");
  if (p->world_size < 1 || p->rank < 0 || p->rank >= p->world_size) return fail(nullptr, SE2M_ERR_INVALID_ARG, "need 0 <= rank < world_size");
  if (p->shard_mode < 0 || p->shard_mode > 2) return fail(nullptr, SE2M_ERR_INVALID_ARG, "shard_mode must be 0, 1 or 2");
  const bool fe_unset = p->fe_z_min == 0 && p->fe_z_max == 0 && p->fe_gate == 0 && p->fe_ray_eps == 0 && p->fe_prior_var == 0;
  if (!fe_unset && (!(p->fe_z_min < p->fe_z_max) || !(p->fe_gate > 0) || !(p->fe_ray_eps >= 0) || !(p->fe_prior_var > 0)))
    return fail(nullptr, SE2M_ERR_INVALID_ARG, "front-end params: need z_min < z_max, gate > 0, ray_eps >= 0, prior_var > 0");
  if (p->inpaint != 0 && p->inpaint != 1) return fail(nullptr, SE2M_ERR_INVALID_ARG, "inpaint must be 0 or 1");
  if (p->chain_segments < 0) return fail(nullptr, SE2M_ERR_INVALID_ARG, "chain_segments must be >= 0");
  if (p->ellipse_ex / p->resolution > 32 || p->ellipse_ey / p->resolution > 32)
    return fail(nullptr, SE2M_ERR_UNSUPPORTED, "footprint radius > 32 cells is not built into this library");
  return SE2M_OK;
}

// Yaw chain: on maps big enough that every CTA takes all its bins, the moments are carried
// along the bins in S segments (restart at each segment bound floor(H s / S)); small maps split the bins
// across CTAs instead (S = H: no chain).  S does not depend on yaw sharding: a yaw shard whose first bin is
// not a segment bound replays the chain from its segment's bound without storing (AssessParams::k_store), so
// every state's FP32 arithmetic — and result — is the unsharded map's, bit for bit (pin Q13).  requested:
// params.chain_segments (0 = auto: SE2M_SEGMENTS_LARGE_R segments for footprint radii R_T >= 16, where the
// chain restarts are cheap next to the per-bin moments and the balanced shards of G = 2, 4, 8 ranks then
// start on segment bounds, else SE2M_SEGMENTS segments).
#ifndef SE2M_SEGMENTS
#define SE2M_SEGMENTS 1        // one chain over all representative bins (A/B on the large map: DESIGN.md §7)
#endif
#ifndef SE2M_SEGMENTS_LARGE_R
#define SE2M_SEGMENTS_LARGE_R 8
#endif
#ifndef SE2M_BORDER_ROWS_EDGE
#define SE2M_BORDER_ROWS_EDGE 0  // the top / bottom border tile rows with the edge chain as side launches on the
                                 // edge stream: measured 1.127 vs 1.048 ms (large, bench conditions) — off
#endif
#ifndef SE2M_MAIN_FIRST
#define SE2M_MAIN_FIRST 1      // launch order of the main / edge assess kernels on one-wave grids (AssessParams::main_first)
#endif
#ifndef SE2M_EDGE_SEGMENTS
#define SE2M_EDGE_SEGMENTS 4   // the vertical-window-edge kernel's chain: at least this many segments
#endif
static int chain_segments(int H, long long cells, int R_T, int requested) {
  if (H < 18 || cells < 512LL * 512LL) return H;
  if (requested > 0) return std::min(H, requested);
  return std::min(H, R_T >= 16 ? SE2M_SEGMENTS_LARGE_R : SE2M_SEGMENTS);
}

// Yaw shards: rank g of G owns the representative bins [H g / G, H (g + 1) / G) (balanced, contiguous).
static void yaw_share(int H, int rank, int G, int* lo, int* hi) {
  *lo = (int)((long long)H * rank / G);
  *hi = (int)((long long)H * (rank + 1) / G);
}

// The chain tables of one segment must fit a CTA's shared memory next to the tile planes (the launch splits
// the bins of a CTA only at segment bounds): large footprints fall back to more, shorter segments.
// Decided against the B200 opt-in limit (227 KB) so that the host-only shard plan agrees with init.
constexpr size_t kSmemOptinB200 = 227 * 1024;
static int seg_table_cap(const se2m_map* m, int s_lo, int s_hi) {  // run entries of segments [s_lo, s_hi)
  const int kb = seg_bound(m->H, m->seg, s_lo), ke = seg_bound(m->H, m->seg, s_hi);
  const int nf = m->full_off[ke] - m->full_off[kb], nc = m->chain_off[ke] - m->chain_off[kb];
  return std::max(1, chain_border(m->R_T) ? nf + nc : std::max(nf, nc));
}
static void tables_for_segments(se2m_map* m, const std::vector<int4>& runs, const std::vector<int>& nrows, int S,
                                std::vector<int4>& full, std::vector<int4>& chain) {
  for (;;) {
    m->seg = S;
    full.clear();
    chain.clear();
    build_tables(m, runs, nrows, full, chain);
    if (S >= m->H) return;
    int cap = 1, bins = 1;
    for (int q = 0; q < S; ++q) {
      cap = std::max(cap, seg_table_cap(m, q, q + 1));
      bins = std::max(bins, seg_bound(m->H, S, q + 1) - seg_bound(m->H, S, q));
    }
    if (assess_smem_bytes(m->R_T, cap, bins) <= kSmemOptinB200) return;
    S = std::min(m->H, 2 * S);
  }
}

extern "C" se2m_status se2m_shard_plan(const se2m_params* p, int32_t* n_rep, int32_t* k_lo, int32_t* k_hi,
                                       int32_t* tile_y, int32_t* row_mod, int32_t* row_rank) {
  se2m_status st = validate(p);
  if (st != SE2M_OK) return st;
  se2m_map m;  // host-only: no device memory, no CUDA calls
  m.prm = *p;
  m.paired = (p->n_yaw % 2 == 0) ? 1 : 0;
  m.H = m.paired ? p->n_yaw / 2 : p->n_yaw;
  std::vector<int4> runs;
  std::vector<int> nrows;
  std::vector<float4> geo, geoc;
  std::vector<float2> cs;
  if (!build_stencils(&m, runs, nrows, geo, geoc, cs)) return fail(nullptr, SE2M_ERR_UNSUPPORTED, "stencil");
  const bool yaw = p->shard_mode == SE2M_SHARD_YAW && p->world_size > 1;
  const bool rows = p->shard_mode == SE2M_SHARD_ROWS && p->world_size > 1;
  if (n_rep) *n_rep = m.H;
  int lo = 0, hi = m.H;
  if (yaw) yaw_share(m.H, p->rank, p->world_size, &lo, &hi);
  if (k_lo) *k_lo = lo;
  if (k_hi) *k_hi = hi;
  if (tile_y) *tile_y = tile_rows(m.R_T);
  if (row_mod) *row_mod = rows ? p->world_size : 1;
  if (row_rank) *row_rank = rows ? p->rank : 0;
  return SE2M_OK;
}

// ---- row-band halo exchange (SE2M_SHARD_ROWS) --------------------
// Rank g owns the world tile rows TJ = g (mod G).  Assessing tile row TJ reads R_T rows on either side
// (the CTA's halo), which lie in tile rows TJ - 1 (rank g - 1) and TJ + 1 (rank g + 1) when R_T <= TY.
// A rank that received only its own rows sends, for every owned tile row, its first R_T rows to rank
// g - 1 and its last R_T rows to rank g + 1.  Both sides enumerate the slabs from the common window
// origin (every rank shifts the same window), so no metadata is exchanged; the list has a fixed
// capacity per window size so the buffers are allocated once.
static int halo_cap(int ny, int TY, int G) { return ((ny + TY - 1) / TY + 3 + G - 1) / G; }
// tile rows sent by `sender`: TJ0, TJ0 + G, ... <= TJb (the tile rows meeting the window, +-1)
static void halo_list(long long J_M, int ny, int TY, int G, int sender, long long* TJ0, long long* TJb) {
  const long long TJa = floor_div(J_M, TY) - 1;
  *TJb = floor_div(J_M + ny - 1, TY) + 1;
  *TJ0 = TJa + pmod((long long)sender - TJa, G);
}
static se2m_status halo_check(const se2m_params* p, int R_T) {
  if (p->shard_mode != SE2M_SHARD_ROWS || p->world_size < 2)
    return SE2M_ERR_INVALID_ARG;
  if (R_T > tile_rows(R_T)) return SE2M_ERR_UNSUPPORTED;  // the halo would reach tile rows TJ +- 2
  return SE2M_OK;
}

extern "C" se2m_status se2m_halo_plan(const se2m_params* p, int64_t J_M, int32_t sender, int32_t last, int32_t* cap,
                                      int32_t* slab_rows, int64_t* first_rows) {
  se2m_status st = validate(p);
  if (st != SE2M_OK) return st;
  se2m_map m;  // host-only: the footprint radius decides R_T and the tile height
  m.prm = *p;
  m.paired = (p->n_yaw % 2 == 0) ? 1 : 0;
  m.H = m.paired ? p->n_yaw / 2 : p->n_yaw;
  std::vector<int4> runs;
  std::vector<int> nrows;
  std::vector<float4> geo, geoc;
  std::vector<float2> cs;
  if (!build_stencils(&m, runs, nrows, geo, geoc, cs)) return fail(nullptr, SE2M_ERR_UNSUPPORTED, "stencil");
  st = halo_check(p, m.R_T);
  if (st != SE2M_OK) return fail(nullptr, st, "halo_plan: needs SE2M_SHARD_ROWS, world_size > 1, R_T <= tile rows");
  if (sender < 0 || sender >= p->world_size) return fail(nullptr, SE2M_ERR_INVALID_ARG, "halo_plan: bad sender");
  const int TY = tile_rows(m.R_T), G = p->world_size, n = halo_cap(p->ny, TY, G);
  if (cap) *cap = n;
  if (slab_rows) *slab_rows = m.R_T;
  if (first_rows) {
    long long TJ0, TJb;
    halo_list(J_M, p->ny, TY, G, sender, &TJ0, &TJb);
    for (int q = 0; q < n; ++q) {
      const long long TJ = TJ0 + (long long)q * G;
      first_rows[q] = TJ <= TJb ? TJ * TY + (last ? TY - m.R_T : 0) : INT64_MIN;
    }
  }
  return SE2M_OK;
}

extern "C" se2m_status se2m_init(const se2m_params* p, se2m_map** out) {
  if (!out) return fail(nullptr, SE2M_ERR_INVALID_ARG, "out is NULL");
  se2m_status st = validate(p);
  if (st != SE2M_OK) return st;
  se2m_map* m = new (std::nothrow) se2m_map();
  if (!m) return fail(nullptr, SE2M_ERR_OOM, "host allocation failed");
  m->prm = *p;
  if (m->prm.fe_z_min == 0 && m->prm.fe_z_max == 0 && m->prm.fe_gate == 0 && m->prm.fe_ray_eps == 0 &&
      m->prm.fe_prior_var == 0) {  // front-end block left zero: the documented defaults
    m->prm.fe_z_min = -1.5; m->prm.fe_z_max = 1.5; m->prm.fe_gate = 2.0; m->prm.fe_ray_eps = 0.05;
    m->prm.fe_prior_var = 1e-4;
  }
  auto bail = [&](se2m_status s) {
    g_init_error = m->err;
    se2m_destroy(m);
    return s;
  };
  int n_dev = 0;
  cudaError_t e = cudaGetDeviceCount(&n_dev);
  if (e != cudaSuccess) { cuda_fail(m, e, "cudaGetDeviceCount"); return bail(SE2M_ERR_CUDA); }
  if (p->device < 0 || p->device >= n_dev) { fail(m, SE2M_ERR_INVALID_ARG, "device ordinal out of range"); return bail(SE2M_ERR_INVALID_ARG); }
  DevGuard dev_guard_(p->device);
  if (p->cuda_stream) m->stream = (cudaStream_t)p->cuda_stream;
  else {
    e = cudaStreamCreateWithFlags(&m->stream, cudaStreamNonBlocking);
    if (e != cudaSuccess) { cuda_fail(m, e, "cudaStreamCreate"); return bail(SE2M_ERR_CUDA); }
    m->own_stream = true;
  }
  const int n = p->n_yaw;
  m->paired = (n % 2 == 0) ? 1 : 0;
  m->H = m->paired ? n / 2 : n;
  m->k_lo = 0; m->k_hi = m->H;
  std::vector<int4> runs;
  std::vector<int> nrows;
  std::vector<float4> geo, geoc;
  std::vector<float2> cs;
  if (!build_stencils(m, runs, nrows, geo, geoc, cs)) {
    fail(m, SE2M_ERR_UNSUPPORTED, "footprint stencil could not be built (radius or shape)");
    return bail(SE2M_ERR_UNSUPPORTED);
  }
  const bool yaw_sharded = p->shard_mode == SE2M_SHARD_YAW && p->world_size > 1;
  std::vector<int4> full, chain;
  tables_for_segments(m, runs, nrows, chain_segments(m->H, (long long)p->nx * p->ny, m->R_T, p->chain_segments), full,
                      chain);
  if (yaw_sharded) yaw_share(m->H, p->rank, p->world_size, &m->k_lo, &m->k_hi);
  // Eq. 4 (reading R6/R7): window origin = floor(x/r) - nx/2 in IEEE double
  m->I_M = (long long)floor(p->robot_x / p->resolution) - p->nx / 2;
  m->J_M = (long long)floor(p->robot_y / p->resolution) - p->ny / 2;
  m->ldh = (p->nx + 3) / 4 * 4;
  m->trav_words = (p->nx + 31) / 32 + 1;  // world 32-groups of the window map to distinct words
  const size_t plane = (size_t)p->nx * p->ny;
  const size_t nst = plane * n;
  struct { void** ptr; size_t bytes; const char* what; } allocs[] = {
      {(void**)&m->d_h, (size_t)m->ldh * p->ny * 4, "heights"},
      {(void**)&m->d_var, (size_t)m->ldh * p->ny * 4, "variances"},
      {(void**)&m->d_out, nst * sizeof(float4), "state records"},
      {(void**)&m->d_trav, (size_t)n * p->ny * m->trav_words * 4, "trav"},
      {(void**)&m->d_full, std::max<size_t>(1, full.size()) * sizeof(int4), "full table"},
      {(void**)&m->d_full_fmt, std::max<size_t>(1, full.size()) * sizeof(int4), "full table (kernel format)"},
      {(void**)&m->d_full_off, m->full_off.size() * sizeof(int), "full offsets"},
      {(void**)&m->d_chain, std::max<size_t>(1, chain.size()) * sizeof(int4), "chain table"},
      {(void**)&m->d_chain_off, m->chain_off.size() * sizeof(int), "chain offsets"},
      {(void**)&m->d_chain_mid, m->chain_mid.size() * sizeof(int), "chain cell offsets"},
      {(void**)&m->d_geo, geo.size() * sizeof(float4), "geo"},
      {(void**)&m->d_geoc, geoc.size() * sizeof(float4), "geoc"},
      {(void**)&m->d_cs, cs.size() * sizeof(float2), "cs"},
      {(void**)&m->d_segb, (size_t)(m->seg + 1) * sizeof(int), "segment bounds"},
      {(void**)&m->d_seg_rst, (size_t)m->H, "restart flags"},
  };
  for (auto& a : allocs) {
    e = cudaMalloc(a.ptr, a.bytes);
    if (e != cudaSuccess) {
      fail(m, e == cudaErrorMemoryAllocation ? SE2M_ERR_OOM : SE2M_ERR_CUDA, std::string("cudaMalloc(") + a.what + ")");
      return bail(e == cudaErrorMemoryAllocation ? SE2M_ERR_OOM : SE2M_ERR_CUDA);
    }
  }
  // the full rows in the kernel's run-entry format: byte offsets into {P0, P2} (8 B) and PX (4 B), float dj
  std::vector<int4> full_fmt(full.size());
  for (size_t q = 0; q < full.size(); ++q) {
    const float dj = (float)(full[q].z - m->R_T);
    int dji;
    memcpy(&dji, &dj, 4);
    full_fmt[q] = make_int4(full[q].x * 8, full[q].y * 8, full[q].x * 4, dji);
  }
  std::vector<int> segb(m->seg + 1);
  std::vector<unsigned char> seg_rst(m->H);
  for (int q = 0; q <= m->seg; ++q) segb[q] = seg_bound(m->H, m->seg, q);
  for (int k = 0; k < m->H; ++k) seg_rst[k] = seg_restart(m->H, m->seg, k) ? 1 : 0;
  if ((e = cudaMemcpyAsync(m->d_segb, segb.data(), segb.size() * sizeof(int), cudaMemcpyHostToDevice, m->stream)) ||
      (e = cudaMemcpyAsync(m->d_seg_rst, seg_rst.data(), seg_rst.size(), cudaMemcpyHostToDevice, m->stream)) ||
      (e = cudaMemcpyAsync(m->d_full, full.data(), full.size() * sizeof(int4), cudaMemcpyHostToDevice, m->stream)) ||
      (e = cudaMemcpyAsync(m->d_full_fmt, full_fmt.data(), full_fmt.size() * sizeof(int4), cudaMemcpyHostToDevice, m->stream)) ||
      (e = cudaMemcpyAsync(m->d_full_off, m->full_off.data(), m->full_off.size() * sizeof(int), cudaMemcpyHostToDevice, m->stream)) ||
      (e = cudaMemcpyAsync(m->d_chain, chain.data(), chain.size() * sizeof(int4), cudaMemcpyHostToDevice, m->stream)) ||
      (e = cudaMemcpyAsync(m->d_chain_off, m->chain_off.data(), m->chain_off.size() * sizeof(int), cudaMemcpyHostToDevice, m->stream)) ||
      (e = cudaMemcpyAsync(m->d_chain_mid, m->chain_mid.data(), m->chain_mid.size() * sizeof(int), cudaMemcpyHostToDevice, m->stream)) ||
      (e = cudaMemcpyAsync(m->d_geo, geo.data(), geo.size() * sizeof(float4), cudaMemcpyHostToDevice, m->stream)) ||
      (e = cudaMemcpyAsync(m->d_geoc, geoc.data(), geoc.size() * sizeof(float4), cudaMemcpyHostToDevice, m->stream)) ||
      (e = cudaMemcpyAsync(m->d_cs, cs.data(), cs.size() * sizeof(float2), cudaMemcpyHostToDevice, m->stream)) ||
      (e = cudaMemsetAsync(m->d_h, 0xff, (size_t)m->ldh * p->ny * 4, m->stream)) ||  // 0xffffffff = NaN: unknown
      (e = cudaMemsetAsync(m->d_var, 0, (size_t)m->ldh * p->ny * 4, m->stream)) ||
      (e = cudaMemsetAsync(m->d_trav, 0, (size_t)n * p->ny * m->trav_words * 4, m->stream)) ||
      (e = cudaStreamSynchronize(m->stream))) {
    cuda_fail(m, e, "init upload");
    return bail(SE2M_ERR_CUDA);
  }
  if (p->nccl_unique_id && p->world_size > 1) {  // the row-band halo transport (collective over the ranks)
    const NcclApi& nc = nccl_api();
    if (!nc.ok) { fail(m, SE2M_ERR_NCCL, "NCCL: " + nc.err); return bail(SE2M_ERR_NCCL); }
    ncclUniqueId id;
    memcpy(&id, p->nccl_unique_id, sizeof id);
    const ncclResult_t r = nc.CommInitRank(&m->comm, p->world_size, id, p->rank);
    if (r != ncclSuccess) {
      m->comm = nullptr;
      fail(m, SE2M_ERR_NCCL, std::string("ncclCommInitRank: ") + nc.GetErrorString(r));
      return bail(SE2M_ERR_NCCL);
    }
  }
  m->prm.nccl_unique_id = nullptr;  // copied (the caller's pointer need not outlive se2m_init)
  {  // the vertical-window-edge kernel's yaw chain (its own segments; see se2m_map::seg_e)
    const bool edge_kernel = tile_rows(m->R_T) == 32 && chain_border(m->R_T);
    m->seg_e = (edge_kernel && m->seg < m->H) ? std::min(m->H, std::max(m->seg, SE2M_EDGE_SEGMENTS)) : m->seg;
    if (m->seg_e == m->seg) {
      m->chain_off_e = m->chain_off; m->chain_mid_e = m->chain_mid;
      m->d_chain_e = m->d_chain; m->d_chain_off_e = m->d_chain_off; m->d_chain_mid_e = m->d_chain_mid;
      m->d_segb_e = m->d_segb; m->d_seg_rst_e = m->d_seg_rst;
    } else {
      std::vector<int4> chain_e;
      build_chain(m, runs, nrows, m->seg_e, chain_e, m->chain_off_e, m->chain_mid_e);
      std::vector<int> segb_e(m->seg_e + 1);
      std::vector<unsigned char> rst_e(m->H);
      for (int q = 0; q <= m->seg_e; ++q) segb_e[q] = seg_bound(m->H, m->seg_e, q);
      for (int k = 0; k < m->H; ++k) rst_e[k] = seg_restart(m->H, m->seg_e, k) ? 1 : 0;
      m->own_edge_tables = true;
      if ((e = cudaMalloc(&m->d_chain_e, std::max<size_t>(1, chain_e.size()) * sizeof(int4))) ||
          (e = cudaMalloc(&m->d_chain_off_e, m->chain_off_e.size() * sizeof(int))) ||
          (e = cudaMalloc(&m->d_chain_mid_e, m->chain_mid_e.size() * sizeof(int))) ||
          (e = cudaMalloc(&m->d_segb_e, segb_e.size() * sizeof(int))) ||
          (e = cudaMalloc(&m->d_seg_rst_e, rst_e.size())) ||
          (e = cudaMemcpyAsync(m->d_chain_e, chain_e.data(), chain_e.size() * sizeof(int4), cudaMemcpyHostToDevice, m->stream)) ||
          (e = cudaMemcpyAsync(m->d_chain_off_e, m->chain_off_e.data(), m->chain_off_e.size() * sizeof(int), cudaMemcpyHostToDevice, m->stream)) ||
          (e = cudaMemcpyAsync(m->d_chain_mid_e, m->chain_mid_e.data(), m->chain_mid_e.size() * sizeof(int), cudaMemcpyHostToDevice, m->stream)) ||
          (e = cudaMemcpyAsync(m->d_segb_e, segb_e.data(), segb_e.size() * sizeof(int), cudaMemcpyHostToDevice, m->stream)) ||
          (e = cudaMemcpyAsync(m->d_seg_rst_e, rst_e.data(), rst_e.size(), cudaMemcpyHostToDevice, m->stream)) ||
          (e = cudaStreamSynchronize(m->stream))) {
        cuda_fail(m, e, "edge chain tables");
        return bail(SE2M_ERR_CUDA);
      }
    }
  }
  m->tma_ok = make_tensor_map(m, &m->tmap, m->d_h);
  {
    int optin = 0;
    if (cudaDeviceGetAttribute(&optin, cudaDevAttrMaxSharedMemoryPerBlockOptin, p->device) == cudaSuccess && optin > 0)
      m->smem_optin = optin;
    int nsm = 0;
    if (cudaDeviceGetAttribute(&nsm, cudaDevAttrMultiProcessorCount, p->device) == cudaSuccess && nsm > 0) m->n_sm = nsm;
  }
  *out = m;
  return SE2M_OK;
}

extern "C" void se2m_destroy(se2m_map* m) {
  if (!m) return;
  DevGuard dev_guard_(m->prm.device);
  if (m->stream) cudaStreamSynchronize(m->stream);
  void* ptrs[] = {m->d_sdf, m->d_var, m->d_pts, m->fe.key, m->fe.idx, m->fe.skey, m->fe.sidx, m->fe.meas,
                  m->fe.counts, m->fe.bbox, m->fe.temp, m->d_h, m->d_out, m->d_trav, m->d_full, m->d_full_fmt, m->d_segb, m->d_seg_rst, m->d_full_off, m->d_chain, m->d_chain_off, m->d_chain_mid, m->d_geo, m->d_geoc,
                  m->d_cs, m->d_stage, m->d_qxyt, m->d_qout, m->d_qcnt, m->d_hin, m->d_site, m->d_ipc, m->d_sdf_g};
  for (void* q : ptrs)
    if (q) cudaFree(q);
  if (m->h_ipc) cudaFreeHost(m->h_ipc);
  if (m->copy_stream) {
    cudaStreamSynchronize(m->copy_stream);
    cudaStreamDestroy(m->copy_stream);
  }
  for (int b = 0; b < 2; ++b) {
    if (m->d_rep[b]) cudaFree(m->d_rep[b]);
    if (m->ev_gathered[b]) cudaEventDestroy(m->ev_gathered[b]);
    if (m->ev_copied[b]) cudaEventDestroy(m->ev_copied[b]);
  }
  if (m->edge_stream) {
    cudaStreamSynchronize(m->edge_stream);
    cudaStreamDestroy(m->edge_stream);
  }
  if (m->ev_fork) cudaEventDestroy(m->ev_fork);
  if (m->ev_join) cudaEventDestroy(m->ev_join);
  for (float* b : m->d_halo)
    if (b) cudaFree(b);
  if (m->own_edge_tables) {
    void* e_ptrs[] = {m->d_chain_e, m->d_chain_off_e, m->d_chain_mid_e, m->d_segb_e, m->d_seg_rst_e};
    for (void* q : e_ptrs)
      if (q) cudaFree(q);
  }
  if (m->comm) nccl_api().CommDestroy(m->comm);  // after the stream drained: no transfer in flight
  if (m->step_exec) cudaGraphExecDestroy(m->step_exec);
  if (m->own_stream && m->stream) cudaStreamDestroy(m->stream);
  delete m;
}

extern "C" se2m_status se2m_update_elevation(se2m_map* m, int32_t i0, int32_t j0, int32_t w, int32_t h,
                                             const float* heights, int64_t ld, const uint8_t* known, int32_t mem) {
  SE2M_ENTER(m);
  if (w == 0 || h == 0) return SE2M_OK;  // nothing to write (the pointer of an empty array may be NULL)
  if (!heights || w < 0 || h < 0 || ld < w || (mem != SE2M_MEM_HOST && mem != SE2M_MEM_DEVICE))
    return fail(m, SE2M_ERR_INVALID_ARG, "update_elevation: bad pointer / size / mem");
  if (i0 < 0 || j0 < 0 || (long long)i0 + w > m->prm.nx || (long long)j0 + h > m->prm.ny)
    return fail(m, SE2M_ERR_OUT_OF_RANGE, "update_elevation: rectangle outside the window");
  if (w == 0 || h == 0) return SE2M_OK;
  const float* src = heights;
  const uint8_t* kn = known;
  long long sld = ld;
  if (mem == SE2M_MEM_HOST) {
    const size_t hb = (size_t)w * h * 4, kb = known ? (size_t)w * h : 0;
    se2m_status st = ensure_stage(m, hb + kb);
    if (st != SE2M_OK) return st;
    float* dh = m->d_stage;
    CUDA_TRY(m, cudaMemcpy2DAsync(dh, (size_t)w * 4, heights, (size_t)ld * 4, (size_t)w * 4, h, cudaMemcpyHostToDevice, m->stream), "H2D heights");
    if (known) {
      uint8_t* dk = reinterpret_cast<uint8_t*>(m->d_stage) + hb;
      CUDA_TRY(m, cudaMemcpy2DAsync(dk, (size_t)w, known, (size_t)ld, (size_t)w, h, cudaMemcpyHostToDevice, m->stream), "H2D known");
      kn = dk;
    }
    src = dh;
    sld = w;
  }
  const int px0 = pmod(m->I_M + i0, m->prm.nx), py0 = pmod(m->J_M + j0, m->prm.ny);
  CUDA_TRY(m, launch_scatter_rect(m->d_h, m->d_var, (float)m->prm.fe_prior_var, m->ldh, m->prm.nx, m->prm.ny, px0, py0,
                                  w, h, src, sld, kn, m->stream), "scatter");
  m->launches++;
  m->have_data = true;
  m->inpaint_valid = false;
  m->dirty.push_back(Rect{m->I_M + i0, m->I_M + i0 + w, m->J_M + j0, m->J_M + j0 + h});
  return SE2M_OK;
}

// Eq. 4 recentre shared by se2m_shift_window and se2m_step: moves the origin, records the dirty strips
// (H9) and returns the logical rectangles (i0, j0, w, h) of the window that entered (n_strips <= 2;
// *all = the whole window was replaced).  Launches nothing.
static void recentre(se2m_map* m, double x, double y, long long* pdi, long long* pdj, int4 strips[2],
                     int* n_strips, bool* all) {
  const int nx = m->prm.nx, ny = m->prm.ny;
  // Eq. 4: p_M = l_res * floor(x / l_res); window origin = floor(x/r) - nx/2
  const long long I_M = (long long)floor(x / m->prm.resolution) - nx / 2;
  const long long J_M = (long long)floor(y / m->prm.resolution) - ny / 2;
  const long long di = I_M - m->I_M, dj = J_M - m->J_M;
  *pdi = di; *pdj = dj; *n_strips = 0; *all = false;
  if (di == 0 && dj == 0) return;
  const Rect old_w{m->I_M, m->I_M + nx, m->J_M, m->J_M + ny};
  const Rect new_w{I_M, I_M + nx, J_M, J_M + ny};
  m->I_M = I_M;
  m->J_M = J_M;
  m->inpaint_valid = false;
  m->sdf_valid = false;  // the SDF layers are in ring order of the old window's risk map
  if (std::llabs(di) >= nx || std::llabs(dj) >= ny) {  // displacement >= side: every cell leaves
    *all = true;
    strips[0] = make_int4(0, 0, nx, ny);
    *n_strips = 1;
    m->all_dirty = true;
    m->dirty.clear();
    return;
  }
  // column strip: logical columns [nx - di, nx) if di > 0, [0, -di) if di < 0, all rows; row strip alike
  if (di != 0) {
    const int w = (int)std::llabs(di);
    strips[(*n_strips)++] = make_int4(di > 0 ? nx - w : 0, 0, w, ny);
  }
  if (dj != 0) {
    const int hgt = (int)std::llabs(dj);
    strips[(*n_strips)++] = make_int4(0, dj > 0 ? ny - hgt : 0, nx, hgt);
  }
  // dirty: the entered strips of the new window and the vacated strips of the old one (H9)
  if (di > 0) { m->dirty.push_back(Rect{old_w.I1, new_w.I1, new_w.J0, new_w.J1}); m->dirty.push_back(Rect{old_w.I0, new_w.I0, old_w.J0, old_w.J1}); }
  if (di < 0) { m->dirty.push_back(Rect{new_w.I0, old_w.I0, new_w.J0, new_w.J1}); m->dirty.push_back(Rect{new_w.I1, old_w.I1, old_w.J0, old_w.J1}); }
  if (dj > 0) { m->dirty.push_back(Rect{new_w.I0, new_w.I1, old_w.J1, new_w.J1}); m->dirty.push_back(Rect{old_w.I0, old_w.I1, old_w.J0, new_w.J0}); }
  if (dj < 0) { m->dirty.push_back(Rect{new_w.I0, new_w.I1, new_w.J0, old_w.J0}); m->dirty.push_back(Rect{old_w.I0, old_w.I1, new_w.J1, old_w.J1}); }
}

static void clamp_out(long long d, int32_t* out) {
  if (out) *out = (int32_t)std::max<long long>(INT32_MIN, std::min<long long>(INT32_MAX, d));
}

extern "C" se2m_status se2m_shift_window(se2m_map* m, double x, double y, int32_t* out_di, int32_t* out_dj) {
  SE2M_ENTER(m);
  if (!isfinite(x) || !isfinite(y)) return fail(m, SE2M_ERR_INVALID_ARG, "shift_window: position not finite");
  long long di, dj;
  int4 strips[2];
  int ns;
  bool all;
  recentre(m, x, y, &di, &dj, strips, &ns, &all);
  clamp_out(di, out_di);
  clamp_out(dj, out_dj);
  if (ns == 0) return SE2M_OK;
  // cells entering the window (their slots held cells that left): unknown — both strips in one launch (the strip
  // fill of se2m_step with an empty world: every cell NaN, variances untouched)
  FillArgs f;
  memset(&f, 0, sizeof f);
  f.h = m->d_h; f.var = nullptr; f.ldh = m->ldh;
  f.nx = m->prm.nx; f.ny = m->prm.ny; f.pxM = pmod(m->I_M, f.nx); f.pyM = pmod(m->J_M, f.ny);
  f.I_M = m->I_M; f.J_M = m->J_M;
  f.world = nullptr; f.ww = 0; f.wh = 0;
  f.n = ns;
  for (int q = 0; q < ns; ++q) f.rect[q] = strips[q];
  CUDA_TRY(m, launch_fill_strips(f, m->stream), "clear");
  m->launches++;
  return SE2M_OK;
}

// The vertical-window-edge kernel's stream.  SE2M_EDGE_PRIORITY = 1 creates it at the device's greatest priority
// (the block scheduler then hands freed SM slots to its CTAs first): measured slower on the large map (1.032 vs
// 1.023 ms, profiles/r02_ab.md), so off.
#ifndef SE2M_EDGE_PRIORITY
#define SE2M_EDGE_PRIORITY 0
#endif
static cudaError_t create_edge_stream(cudaStream_t* s) {
  int lo = 0, hi = 0;
  if (SE2M_EDGE_PRIORITY && cudaDeviceGetStreamPriorityRange(&lo, &hi) == cudaSuccess)
    return cudaStreamCreateWithPriority(s, cudaStreamNonBlocking, hi);
  cudaGetLastError();
  return cudaStreamCreateWithFlags(s, cudaStreamNonBlocking);
}

extern "C" se2m_status se2m_step(se2m_map* m, double x, double y, const float* world, int64_t world_ld,
                                 int64_t world_I0, int64_t world_J0, int32_t world_w, int32_t world_h,
                                 int32_t mem, int32_t* out_di, int32_t* out_dj) {
  SE2M_ENTER(m);
  if (!isfinite(x) || !isfinite(y)) return fail(m, SE2M_ERR_INVALID_ARG, "step: position not finite");
  if (!world || mem != SE2M_MEM_DEVICE || world_w < 0 || world_h < 0 || world_ld < world_w)
    return fail(m, SE2M_ERR_INVALID_ARG, "step: world must be a device plane with ld >= w");
  long long di, dj;
  int4 strips[2];
  int ns;
  bool all;
  recentre(m, x, y, &di, &dj, strips, &ns, &all);
  clamp_out(di, out_di);
  clamp_out(dj, out_dj);
  FillArgs f;
  if (ns > 0) {
    f.h = m->d_h; f.var = m->d_var; f.prior_var = (float)m->prm.fe_prior_var; f.ldh = m->ldh;
    f.nx = m->prm.nx; f.ny = m->prm.ny; f.pxM = pmod(m->I_M, f.nx); f.pyM = pmod(m->J_M, f.ny);
    f.I_M = m->I_M; f.J_M = m->J_M;
    f.world = world; f.world_ld = world_ld; f.wI0 = world_I0; f.wJ0 = world_J0; f.ww = world_w; f.wh = world_h;
    f.n = ns;
    for (int q = 0; q < ns; ++q) f.rect[q] = strips[q];
  }
  // the step's launches: strip fill (H1 + H2), then INCREMENTAL assess (H9)
  auto launches = [&]() -> se2m_status {
    if (ns > 0) {
      CUDA_TRY(m, launch_fill_strips(f, m->stream), "fill strips");
      m->launches++;
      m->have_data = true;
    }
    if (!m->have_data) return SE2M_OK;  // nothing to assess yet
    return se2m_assess_se2(m, SE2M_INCREMENTAL);
  };
  const bool graph = m->prm.step_graph && !m->prm.inpaint && m->step_warm;
  if (!graph) {  // direct launches (the first step also makes the lazy allocations no capture may contain)
    const se2m_status st = launches();
    if (st == SE2M_OK && m->have_data) m->step_warm = true;
    return st;
  }
  if (!m->edge_stream) {  // the assess may fork onto the edge stream: create it outside the capture
    CUDA_TRY(m, create_edge_stream(&m->edge_stream), "cudaStreamCreate(edge)");
    CUDA_TRY(m, cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming), "cudaEventCreate");
    CUDA_TRY(m, cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming), "cudaEventCreate");
  }
  CUDA_TRY(m, cudaStreamBeginCapture(m->stream, cudaStreamCaptureModeThreadLocal), "begin capture");
  const se2m_status st = launches();
  cudaGraph_t g = nullptr;
  const cudaError_t ec = cudaStreamEndCapture(m->stream, &g);
  if (st != SE2M_OK || ec != cudaSuccess || !g) {
    if (g) cudaGraphDestroy(g);
    cudaGetLastError();
    return st != SE2M_OK ? st : cuda_fail(m, ec, "end capture");
  }
  if (m->step_exec) {  // same topology as last step (the usual case): update the kernel parameters in place
    cudaGraphExecUpdateResultInfo info;
    if (cudaGraphExecUpdate(m->step_exec, g, &info) != cudaSuccess) {
      cudaGetLastError();
      cudaGraphExecDestroy(m->step_exec);
      m->step_exec = nullptr;
    }
  }
  cudaError_t e = cudaSuccess;
  if (!m->step_exec) e = cudaGraphInstantiate(&m->step_exec, g, 0);
  if (e == cudaSuccess) e = cudaGraphLaunch(m->step_exec, m->stream);
  cudaGraphDestroy(g);
  if (e != cudaSuccess) return cuda_fail(m, e, "step graph");
  return SE2M_OK;
}


// NEXT-4: (re)compute the inpainted view; cells whose view value changed become dirty.  Synchronises.
static se2m_status run_inpaint(se2m_map* m, int* n_known) {
  const int nx = m->prm.nx, ny = m->prm.ny;
  if (!m->d_hin) {
    CUDA_TRY(m, cudaMalloc(&m->d_hin, (size_t)m->ldh * ny * 4), "cudaMalloc(inpainted view)");
    CUDA_TRY(m, cudaMalloc(&m->d_site, ((size_t)nx * ny + inpaint_seg_ints(nx, ny)) * 4), "cudaMalloc(inpaint scratch)");
    CUDA_TRY(m, cudaMalloc(&m->d_ipc, 8 * sizeof(int)), "cudaMalloc(inpaint counters)");
    CUDA_TRY(m, cudaMallocHost(&m->h_ipc, 8 * sizeof(int)), "cudaMallocHost(inpaint counters)");
    CUDA_TRY(m, cudaMemsetAsync(m->d_hin, 0xff, (size_t)m->ldh * ny * 4, m->stream), "init view");  // NaN
    m->tma_in_ok = m->tma_ok && make_tensor_map(m, &m->tmap_in, m->d_hin);
  }
  CUDA_TRY(m, cudaMemsetAsync(m->d_ipc, 0, sizeof(int), m->stream), "inpaint counters");
  CUDA_TRY(m, launch_inpaint(m->d_h, m->ldh, nx, ny, pmod(m->I_M, nx), pmod(m->J_M, ny), m->d_site, m->d_hin,
                             m->d_ipc, m->d_site + (size_t)nx * ny, m->stream), "inpaint kernels");
  m->launches += 3;
  CUDA_TRY(m, cudaMemcpyAsync(m->h_ipc, m->d_ipc, 5 * sizeof(int), cudaMemcpyDeviceToHost, m->stream), "D2H inpaint");
  CUDA_TRY(m, cudaStreamSynchronize(m->stream), "sync(inpaint)");
  const int* c = m->h_ipc;
  if (c[2] >= 0) m->dirty.push_back(Rect{m->I_M + c[1], m->I_M + c[2] + 1, m->J_M + c[3], m->J_M + c[4] + 1});
  m->inpaint_valid = true;
  if (n_known) *n_known = c[0];
  return SE2M_OK;
}

extern "C" se2m_status se2m_inpaint(se2m_map* m) {
  SE2M_ENTER(m);
  int n_known = 0;
  se2m_status st = run_inpaint(m, &n_known);
  if (st != SE2M_OK) return st;
  if (n_known == 0) return fail(m, SE2M_ERR_STATE, "inpaint: no known cell in the window");
  return SE2M_OK;
}

extern "C" se2m_status se2m_assess_se2(se2m_map* m, int32_t mode) {
  SE2M_ENTER(m);
  if (mode != SE2M_FULL && mode != SE2M_INCREMENTAL) return fail(m, SE2M_ERR_INVALID_ARG, "assess: bad mode");
  if (!m->have_data) return fail(m, SE2M_ERR_STATE, "assess before any update_elevation");
  if (m->prm.inpaint && !m->inpaint_valid) {  // NEXT-4: assess the inpainted view
    se2m_status st = run_inpaint(m, nullptr);
    if (st != SE2M_OK) return st;
  }
  AssessParams p = make_params(m);
  const CUtensorMap* tmap = &m->tmap;
  if (m->prm.inpaint) {
    p.h = m->d_hin;
    tmap = &m->tmap_in;
    p.use_tma = m->tma_in_ok ? 1 : 0;
  }
  const int nx = m->prm.nx, ny = m->prm.ny;
  const int TY = tile_rows(m->R_T);
  // dense grid of world tiles intersecting the window
  const long long TI0 = floor_div(m->I_M, TX), TI1 = floor_div(m->I_M + nx - 1, TX);
  const long long TJ0 = floor_div(m->J_M, TY), TJ1 = floor_div(m->J_M + ny - 1, TY);
  long long gx0 = 0, gx1 = TI1 - TI0 + 1, gy0 = 0, gy1 = TJ1 - TJ0 + 1;  // launch box, tiles rel. to (TI0, TJ0)
  const bool full = mode == SE2M_FULL || m->all_dirty;
  std::vector<int4> rects;
  if (!full) {
    // H9: states within R (Chebyshev bound of every footprint) of a changed cell, as tile rectangles — dilated by
    // R_T >= R: a tile changes kernels (edge / border / main: different rounding) only when the window edge passes
    // within R_T of it, i.e. within R_T of the entered or vacated cells, so INCREMENTAL == FULL bit for bit
    const long long Rd = m->R_T;
    long long bx0 = gx1, bx1 = 0, by0 = gy1, by1 = 0;
    for (const Rect& d : m->dirty) {
      const long long I0 = std::max(d.I0 - Rd, m->I_M), I1 = std::min(d.I1 + Rd, m->I_M + nx);
      const long long J0 = std::max(d.J0 - Rd, m->J_M), J1 = std::min(d.J1 + Rd, m->J_M + ny);
      if (I0 >= I1 || J0 >= J1) continue;
      const int4 t = make_int4((int)(floor_div(I0, TX) - TI0), (int)(floor_div(I1 - 1, TX) - TI0 + 1),
                               (int)(floor_div(J0, TY) - TJ0), (int)(floor_div(J1 - 1, TY) - TJ0 + 1));
      rects.push_back(t);
      bx0 = std::min<long long>(bx0, t.x); bx1 = std::max<long long>(bx1, t.y);
      by0 = std::min<long long>(by0, t.z); by1 = std::max<long long>(by1, t.w);
    }
    if (rects.empty()) { m->dirty.clear(); return SE2M_OK; }  // nothing changed
    if ((int)rects.size() > kMaxRects) rects.assign(1, make_int4((int)bx0, (int)bx1, (int)by0, (int)by1));
    gx0 = bx0; gx1 = bx1; gy0 = by0; gy1 = by1;
    for (int4& t : rects) { t.x -= (int)gx0; t.y -= (int)gx0; t.z -= (int)gy0; t.w -= (int)gy0; }
  }
  p.TI0 = TI0 + gx0; p.TJ0 = TJ0 + gy0;
  p.tiles_x = (int)(gx1 - gx0);
  const int tiles_y = (int)(gy1 - gy0);
  p.n_rects = (int)rects.size();
  for (int q = 0; q < p.n_rects; ++q) p.rects[q] = rects[q];
  p.row_mod = 1; p.row_first = 0;
  if (m->prm.shard_mode == SE2M_SHARD_ROWS && m->prm.world_size > 1) {
    p.row_mod = m->prm.world_size;                       // rank owns world tile rows TJ = rank (mod G)
    p.row_first = pmod((long long)m->prm.rank - p.TJ0, p.row_mod);
  }
  const int grid_rows = tiles_y > p.row_first ? (tiles_y - p.row_first + p.row_mod - 1) / p.row_mod : 0;
  const int n_tiles = p.tiles_x * grid_rows;
  // yaw chunking: all bins per CTA (tile reuse) unless that leaves SMs idle; then split the bins so the
  // CTAs fill one wave (the device's SMs x the kernel's resident CTAs per SM) — each CTA pays the tile
  // load, plane fit and prefix build once, so more, shorter CTAs than that only add fixed cost.  Chunks are
  // whole chain segments (AssessParams::seg): segments [s_a, s_b) cover the launch's bins [k_begin, k_hi).
  const int H = m->H, S = m->seg;
  const int s_a = seg_of(H, S, p.k_begin);
  const int s_b = m->k_hi > p.k_begin ? seg_of(H, S, m->k_hi - 1) + 1 : s_a;
  const int n_seg = s_b - s_a;
  const int nk = m->k_hi - p.k_begin;
  // run tables (and bins) of the largest chunk of c segments: they must fit the CTA's shared memory
  auto chunk_need = [&](int c, int* cap_out, int* bins_out) {
    int cap = 1, bins = 1;
    for (int q = s_a; q < s_b; q += c) {
      const int kb = std::max(p.k_begin, seg_bound(H, S, q)), ke = std::min(m->k_hi, seg_bound(H, S, std::min(S, q + c)));
      const int nf = m->full_off[ke] - m->full_off[kb], nc = m->chain_off[ke] - m->chain_off[kb];
      cap = std::max(cap, chain_border(m->R_T) ? nf + nc : std::max(nf, nc));
      bins = std::max(bins, ke - kb);
    }
    *cap_out = cap;
    *bins_out = bins;
    return assess_smem_bytes(m->R_T, cap, bins);
  };
  if (m->slots_per_sm <= 0 && n_seg > 0) {  // resident CTAs per SM at the whole-range chunk (occupancy API, once)
    int cap0, bins0;
    const size_t sm_full = chunk_need(n_seg, &cap0, &bins0);
    m->slots_per_sm = sm_full <= (size_t)m->smem_optin ? assess_ctas_per_sm(m->R_T, sm_full) : 0;
    if (m->slots_per_sm <= 0) m->slots_per_sm = 2;  // (launch bounds: 2 CTAs of 256 threads per SM)
  }
  int c = std::max(1, n_seg);
  if (n_tiles > 0 && n_seg > 0) {
    const long long slots = (long long)m->n_sm * m->slots_per_sm;
    const long long want_bins = std::max<long long>(1, ((long long)n_tiles * nk + slots - 1) / slots);
    c = (int)std::max<long long>(1, std::min<long long>(n_seg, (want_bins * n_seg + nk - 1) / nk));
  }
  // large footprints take fewer segments per CTA when the tables do not fit
  int cap = 1, bins = 1;
  while (chunk_need(c, &cap, &bins) > (size_t)m->smem_optin && c > 1) c = (c + 1) / 2;
  if (chunk_need(c, &cap, &bins) > (size_t)m->smem_optin)
    return fail(m, SE2M_ERR_UNSUPPORTED, "assess: footprint tables exceed the shared memory of a CTA");
  p.seg_chunk = c;
  p.n_chunks = (n_seg + c - 1) / c;
  p.k_chunk = bins;
  p.tab_cap = cap;
  // vertical-window-edge tile columns (the halo crosses the window's left / right edge): their tiles run
  // in the column-major layout kernel on the edge stream, concurrently (tile_rows == 32 footprints only)
  p.tsplit = 0; p.n_tcols = 0;
  if (tile_rows(m->R_T) == 32 && chain_border(m->R_T) && SE2M_TSPLIT) {
    const int HX = TX + 2 * m->R_T;
    for (int tx = 0; tx < p.tiles_x; ++tx) {
      const long long li0 = (p.TI0 + tx) * TX - m->R_T - m->I_M;
      if (li0 < 0 || li0 + HX > nx) {
        if (p.n_tcols == 4) { p.n_tcols = -1; break; }
        p.tcols[p.n_tcols++] = tx;
      }
    }
    if (p.n_tcols > 0) {
      if (!m->edge_stream) {
        CUDA_TRY(m, create_edge_stream(&m->edge_stream), "cudaStreamCreate(edge)");
        CUDA_TRY(m, cudaEventCreateWithFlags(&m->ev_fork, cudaEventDisableTiming), "cudaEventCreate");
        CUDA_TRY(m, cudaEventCreateWithFlags(&m->ev_join, cudaEventDisableTiming), "cudaEventCreate");
      }
      p.tsplit = 1;
    } else {
      p.n_tcols = 0;
    }
  }
  // the edge kernel's launch: its own yaw chain (seg_e segments, one per CTA when shorter than the main chain)
  AssessParams pe = p;
  if (p.tsplit) {
    const int Se = m->seg_e;
    pe.seg = Se; pe.segb = m->d_segb_e; pe.seg_rst = m->d_seg_rst_e;
    pe.chain = m->d_chain_e; pe.chain_off = m->d_chain_off_e; pe.chain_mid = m->d_chain_mid_e;
    pe.seg_first = seg_of(H, Se, m->k_lo);
    pe.k_begin = seg_bound(H, Se, pe.seg_first);
    const int sa = pe.seg_first, sb = m->k_hi > pe.k_begin ? seg_of(H, Se, m->k_hi - 1) + 1 : sa;
    int ce = Se == m->seg ? p.seg_chunk : 1;
    int cap_e = 1, bins_e = 1;
    for (;;) {
      cap_e = 1; bins_e = 1;
      for (int q = sa; q < sb; q += ce) {
        const int kb = std::max(pe.k_begin, seg_bound(H, Se, q)), ke = std::min(m->k_hi, seg_bound(H, Se, std::min(Se, q + ce)));
        const int nf = m->full_off[ke] - m->full_off[kb], nc = m->chain_off_e[ke] - m->chain_off_e[kb];
        cap_e = std::max(cap_e, nf + nc);  // (edge tiles: chain_border radii only)
        bins_e = std::max(bins_e, ke - kb);
      }
      if (assess_smem_bytes(m->R_T, cap_e, bins_e) <= (size_t)m->smem_optin || ce == 1) break;
      ce = (ce + 1) / 2;
    }
    if (assess_smem_bytes(m->R_T, cap_e, bins_e) > (size_t)m->smem_optin)
      return fail(m, SE2M_ERR_UNSUPPORTED, "assess: footprint tables exceed the shared memory of a CTA (edge)");
    pe.seg_chunk = ce;
    pe.n_chunks = (sb - sa + ce - 1) / ce;
    pe.k_chunk = bins_e;
    pe.tab_cap = cap_e;
  }
  // small grids (both kernels' CTAs fit one wave): the main kernel launches first — its corner / border CTAs
  // are the longest, and with free slots for every CTA the edge kernel loses nothing by starting second
  p.main_first = 0;
  if (p.tsplit && SE2M_MAIN_FIRST) {
    const long long ctas = (long long)p.n_tcols * grid_rows * pe.n_chunks +
                           (long long)(p.tiles_x - p.n_tcols) * grid_rows * p.n_chunks;
    p.main_first = ctas <= (long long)m->n_sm * m->slots_per_sm ? 1 : 0;
  }
  // the window's top / bottom border tile rows (a prefix and a suffix of the grid rows: lj0 grows with the row)
  // run on the edge stream with the edge chain — their general pairs make long CTAs, which shorter chunks
  // keep off the critical path; the main launch covers the middle rows
  AssessParams side[2] = {pe, pe};
  int side_tiles[2] = {0, 0}, n_side = 0;
  AssessParams p0 = p;
  if (p.tsplit && m->seg_e != m->seg && SE2M_BORDER_ROWS_EDGE) {
    const int HY = TY + 2 * m->R_T;
    auto bedge = [&](int gr) {
      const long long lj0 = (p.TJ0 + p.row_first + gr * p.row_mod) * TY - m->R_T - m->J_M;
      return lj0 < 0 || lj0 + HY > ny;
    };
    int pre = 0, suf = 0;
    while (pre < grid_rows && bedge(pre)) ++pre;
    while (suf < grid_rows - pre && bedge(grid_rows - 1 - suf)) ++suf;
    if (pre + suf > 0 && pre + suf < grid_rows) {
      side[0].row_first = p.row_first;                                   // rows [0, pre)
      side[1].row_first = p.row_first + (grid_rows - suf) * p.row_mod;   // rows [grid_rows - suf, grid_rows)
      side_tiles[0] = pre * p.tiles_x;
      side_tiles[1] = suf * p.tiles_x;
      n_side = 2;
      p0.row_first = p.row_first + pre * p.row_mod;                      // the main launch: the middle rows
    }
  }
  if (n_tiles > 0 && n_seg > 0 && m->k_hi > m->k_lo) {
    int nl = 0;
    cudaError_t e = launch_assess(p0, pe, m->R_T, n_tiles, side, side_tiles, n_side, tmap, m->stream, m->edge_stream,
                                  m->ev_fork, m->ev_join, &nl);
    if (e != cudaSuccess) return cuda_fail(m, e, "assess kernel");
    m->launches += nl;
  }
  m->dirty.clear();
  m->all_dirty = false;
  m->sdf_valid = false;  // the SDF follows the risk map: recompute with se2m_compute_sdf
  return SE2M_OK;
}

extern "C" se2m_status se2m_halo_size(const se2m_map* m, int32_t* cap, int32_t* slab_rows) {
  if (!m) return SE2M_ERR_INVALID_ARG;
  const se2m_status st = halo_check(&m->prm, m->R_T);
  if (st != SE2M_OK) return st;
  if (cap) *cap = halo_cap(m->prm.ny, tile_rows(m->R_T), m->prm.world_size);
  if (slab_rows) *slab_rows = m->R_T;
  return SE2M_OK;
}

static HaloArgs halo_args(se2m_map* m, int sender, int last, float* buf, int unpack) {
  HaloArgs a;
  a.h = m->d_h; a.buf = buf; a.ldh = m->ldh; a.nx = m->prm.nx; a.ny = m->prm.ny;
  a.pxM = pmod(m->I_M, a.nx); a.pyM = pmod(m->J_M, a.ny); a.J_M = m->J_M;
  a.G = m->prm.world_size; a.TY = tile_rows(m->R_T); a.R_T = m->R_T; a.last = last; a.unpack = unpack;
  halo_list(m->J_M, a.ny, a.TY, a.G, sender, &a.TJ0, &a.TJb);
  return a;
}

extern "C" se2m_status se2m_halo_pack(se2m_map* m, int32_t dir, float* dst) {
  SE2M_ENTER(m);
  se2m_status st = halo_check(&m->prm, m->R_T);
  if (st != SE2M_OK) return fail(m, st, "halo_pack: needs SE2M_SHARD_ROWS, world_size > 1, R_T <= tile rows");
  if (!dst || (dir != -1 && dir != 1)) return fail(m, SE2M_ERR_INVALID_ARG, "halo_pack: dir must be -1 or +1, dst non-NULL");
  // to rank g - 1: the first R_T rows of each owned tile row; to rank g + 1: the last R_T rows
  const HaloArgs a = halo_args(m, m->prm.rank, dir > 0 ? 1 : 0, dst, 0);
  CUDA_TRY(m, launch_halo(a, halo_cap(a.ny, a.TY, a.G), m->stream), "halo pack");
  m->launches++;
  return SE2M_OK;
}

extern "C" se2m_status se2m_halo_unpack(se2m_map* m, int32_t from, const float* src) {
  SE2M_ENTER(m);
  se2m_status st = halo_check(&m->prm, m->R_T);
  if (st != SE2M_OK) return fail(m, st, "halo_unpack: needs SE2M_SHARD_ROWS, world_size > 1, R_T <= tile rows");
  if (!src || (from != -1 && from != 1)) return fail(m, SE2M_ERR_INVALID_ARG, "halo_unpack: from must be -1 or +1, src non-NULL");
  // slabs from rank g + 1 are the first rows of its tile rows (it packed toward g - 1 = us), from g - 1 the last
  const int G = m->prm.world_size, sender = pmod((long long)m->prm.rank + from, G), last = from < 0 ? 1 : 0;
  const HaloArgs a = halo_args(m, sender, last, const_cast<float*>(src), 1);
  const int cap = halo_cap(a.ny, a.TY, G);
  CUDA_TRY(m, launch_halo(a, cap, m->stream), "halo unpack");
  m->launches++;
  m->have_data = true;
  m->inpaint_valid = false;
  for (int q = 0; q < cap; ++q) {  // written rows are dirty (H9)
    const long long TJ = a.TJ0 + (long long)q * G;
    if (TJ > a.TJb) break;
    const long long W0 = std::max(TJ * a.TY + (last ? a.TY - a.R_T : 0), m->J_M);
    const long long W1 = std::min(TJ * a.TY + (last ? a.TY : a.R_T), m->J_M + a.ny);
    if (W0 < W1) m->dirty.push_back(Rect{m->I_M, m->I_M + a.nx, W0, W1});
  }
  return SE2M_OK;
}

extern "C" se2m_status se2m_exchange_halo(se2m_map* m) {
  SE2M_ENTER(m);
  se2m_status st = halo_check(&m->prm, m->R_T);
  if (st != SE2M_OK) return fail(m, st, "exchange_halo: needs SE2M_SHARD_ROWS, world_size > 1, R_T <= tile rows");
  if (!m->comm) return fail(m, SE2M_ERR_STATE, "exchange_halo: no communicator (params.nccl_unique_id was NULL)");
  const int G = m->prm.world_size, g = m->prm.rank, TY = tile_rows(m->R_T);
  const size_t count = (size_t)halo_cap(m->prm.ny, TY, G) * m->R_T * m->prm.nx;
  for (float*& b : m->d_halo)
    if (!b) CUDA_TRY(m, cudaMalloc(&b, count * sizeof(float)), "cudaMalloc(halo)");
  float *to_lo = m->d_halo[0], *to_hi = m->d_halo[1], *from_hi = m->d_halo[2], *from_lo = m->d_halo[3];
  if ((st = se2m_halo_pack(m, -1, to_lo)) != SE2M_OK) return st;
  if ((st = se2m_halo_pack(m, +1, to_hi)) != SE2M_OK) return st;
  const NcclApi& nc = nccl_api();
  const int lo = (g - 1 + G) % G, hi = (g + 1) % G;
  ncclResult_t r = nc.GroupStart();
  if (r == ncclSuccess) {
    // issue order (send to lo, recv from hi, send to hi, recv from lo) pairs every send with the peer's
    // receive of the same slab set, also when lo == hi (G = 2)
    ncclResult_t q = nc.Send(to_lo, count, ncclFloat32, lo, m->comm, m->stream);
    if (q == ncclSuccess) q = nc.Recv(from_hi, count, ncclFloat32, hi, m->comm, m->stream);
    if (q == ncclSuccess) q = nc.Send(to_hi, count, ncclFloat32, hi, m->comm, m->stream);
    if (q == ncclSuccess) q = nc.Recv(from_lo, count, ncclFloat32, lo, m->comm, m->stream);
    r = nc.GroupEnd();  // always close the group
    if (q != ncclSuccess) r = q;
  }
  if (r != ncclSuccess) return fail(m, SE2M_ERR_NCCL, std::string("halo send/recv: ") + nc.GetErrorString(r));
  m->launches += 1;  // the NCCL group kernel
  if ((st = se2m_halo_unpack(m, +1, from_hi)) != SE2M_OK) return st;
  return se2m_halo_unpack(m, -1, from_lo);
}

extern "C" se2m_status se2m_nccl_unique_id(void* out, int32_t bytes, int32_t* version) {
  if (!out || bytes < (int32_t)sizeof(ncclUniqueId)) return fail(nullptr, SE2M_ERR_INVALID_ARG, "nccl_unique_id: need 128 bytes");
  const NcclApi& nc = nccl_api();
  if (!nc.ok) return fail(nullptr, SE2M_ERR_NCCL, "NCCL: " + nc.err);
  ncclUniqueId id;
  const ncclResult_t r = nc.GetUniqueId(&id);
  if (r != ncclSuccess) return fail(nullptr, SE2M_ERR_NCCL, std::string("ncclGetUniqueId: ") + nc.GetErrorString(r));
  memcpy(out, &id, sizeof id);
  if (version) {
    int v = 0;
    *version = nc.GetVersion(&v) == ncclSuccess ? v : 0;
  }
  return SE2M_OK;
}

extern "C" se2m_status se2m_nccl_selftest(int32_t device, int64_t count, int32_t* version) {
  if (count < 1) return fail(nullptr, SE2M_ERR_INVALID_ARG, "nccl_selftest: count must be >= 1");
  const NcclApi& nc = nccl_api();
  if (!nc.ok) return fail(nullptr, SE2M_ERR_NCCL, "NCCL: " + nc.err);
  DevGuard guard(device);
  int cur = -1;
  if (cudaGetDevice(&cur) != cudaSuccess || cur != device) return fail(nullptr, SE2M_ERR_CUDA, "nccl_selftest: cudaSetDevice");
  if (version) {
    int v = 0;
    *version = nc.GetVersion(&v) == ncclSuccess ? v : 0;
  }
  std::vector<float> sent((size_t)count), got((size_t)count, 0.f);
  for (int64_t i = 0; i < count; ++i) sent[(size_t)i] = (float)((i * 2654435761LL) % 1000003) * 0.5f - 7.25f;
  ncclUniqueId id;
  ncclComm_t comm = nullptr;
  cudaStream_t st = nullptr;
  float *a = nullptr, *b = nullptr;
  std::string err;
  se2m_status rc = SE2M_OK;
  auto cu = [&](cudaError_t e, const char* what) {
    if (e != cudaSuccess && rc == SE2M_OK) { rc = SE2M_ERR_CUDA; err = std::string(what) + ": " + cudaGetErrorString(e); }
    return rc == SE2M_OK;
  };
  auto nk = [&](ncclResult_t r, const char* what) {
    if (r != ncclSuccess && rc == SE2M_OK) { rc = SE2M_ERR_NCCL; err = std::string(what) + ": " + nc.GetErrorString(r); }
    return rc == SE2M_OK;
  };
  const size_t bytes = (size_t)count * sizeof(float);
  if (nk(nc.GetUniqueId(&id), "ncclGetUniqueId") && nk(nc.CommInitRank(&comm, 1, id, 0), "ncclCommInitRank") &&
      cu(cudaStreamCreateWithFlags(&st, cudaStreamNonBlocking), "cudaStreamCreate") &&
      cu(cudaMalloc(&a, bytes), "cudaMalloc") && cu(cudaMalloc(&b, bytes), "cudaMalloc") &&
      cu(cudaMemcpy(a, sent.data(), bytes, cudaMemcpyHostToDevice), "cudaMemcpy") &&
      cu(cudaMemset(b, 0, bytes), "cudaMemset") && nk(nc.GroupStart(), "ncclGroupStart")) {
    ncclResult_t q = nc.Send(a, (size_t)count, ncclFloat32, 0, comm, st);
    if (q == ncclSuccess) q = nc.Recv(b, (size_t)count, ncclFloat32, 0, comm, st);
    const ncclResult_t r = nc.GroupEnd();
    if (nk(q, "ncclSend/ncclRecv") && nk(r, "ncclGroupEnd") && cu(cudaStreamSynchronize(st), "transfer") &&
        cu(cudaMemcpy(got.data(), b, bytes, cudaMemcpyDeviceToHost), "cudaMemcpy") &&
        memcmp(got.data(), sent.data(), bytes) != 0) {
      rc = SE2M_ERR_NCCL;
      err = "the received floats differ from the sent ones";
    }
  }
  if (comm) nc.CommDestroy(comm);
  if (a) cudaFree(a);
  if (b) cudaFree(b);
  if (st) cudaStreamDestroy(st);
  if (rc != SE2M_OK) return fail(nullptr, rc, "nccl_selftest: " + err);
  return SE2M_OK;
}

extern "C" se2m_status se2m_chain_segments(const se2m_map* m, int32_t* segments) {
  if (!m || !segments) return SE2M_ERR_INVALID_ARG;
  *segments = m->seg;
  return SE2M_OK;
}

extern "C" se2m_status se2m_tile_info(const se2m_map* m, int32_t* tile_x, int32_t* tile_y) {
  if (!m) return SE2M_ERR_INVALID_ARG;
  if (tile_x) *tile_x = TX;
  if (tile_y) *tile_y = tile_rows(m->R_T);
  return SE2M_OK;
}


static QueryGeo query_geo(const se2m_map* m) {
  QueryGeo g;
  memset(&g, 0, sizeof g);
  g.r = m->prm.resolution; g.dth = 2.0 * M_PI / m->prm.n_yaw;
  g.I_M = m->I_M; g.J_M = m->J_M;
  g.nx = m->prm.nx; g.ny = m->prm.ny; g.n_yaw = m->prm.n_yaw; g.H = m->H; g.paired = m->paired;
  g.k_lo = m->k_lo; g.k_hi = m->k_hi;
  const bool rows = m->prm.shard_mode == SE2M_SHARD_ROWS && m->prm.world_size > 1;
  g.row_mod = rows ? m->prm.world_size : 1; g.row_rank = rows ? m->prm.rank : 0;
  g.TY = tile_rows(m->R_T); g.trav_words = m->trav_words;
  return g;
}

// Stage n queries on the device; returns the number of output floats per query slot (cap grows).
static se2m_status stage_queries(se2m_map* m, int64_t n, const double* xyt) {
  if ((size_t)n > m->q_cap) {
    if (m->d_qxyt) cudaFree(m->d_qxyt);
    if (m->d_qout) cudaFree(m->d_qout);
    m->d_qxyt = nullptr; m->d_qout = nullptr; m->q_cap = 0;
    CUDA_TRY(m, cudaMalloc(&m->d_qxyt, (size_t)n * 3 * sizeof(double)), "cudaMalloc(query)");
    CUDA_TRY(m, cudaMalloc(&m->d_qout, (size_t)n * 5 * sizeof(float)), "cudaMalloc(query)");
    m->q_cap = (size_t)n;
  }
  if (!m->d_qcnt) CUDA_TRY(m, cudaMalloc(&m->d_qcnt, sizeof(int)), "cudaMalloc(query)");
  CUDA_TRY(m, cudaMemsetAsync(m->d_qcnt, 0, sizeof(int), m->stream), "query counter");
  // host or device xyt (se2m_query_async with SE2M_MEM_DEVICE): the direction comes from the pointer (UVA)
  CUDA_TRY(m, cudaMemcpyAsync(m->d_qxyt, xyt, (size_t)n * 3 * sizeof(double), cudaMemcpyDefault, m->stream),
           "stage query");
  return SE2M_OK;
}

// Pinned (page-locked, device-mapped) host memory is read and written by the query kernels in place (zero copy over
// PCIe: no staging copy in, no D2H copy out — two fewer operations on the map's stream per call); pageable host
// buffers take the staged path.  SE2M_ZERO_COPY = 0: always staged.
#ifndef SE2M_ZERO_COPY
#define SE2M_ZERO_COPY 1
#endif
static void* mapped_host(const void* h) {
  if (!SE2M_ZERO_COPY || !h) return nullptr;
  cudaPointerAttributes a;
  if (cudaPointerGetAttributes(&a, h) != cudaSuccess) {
    cudaGetLastError();
    return nullptr;
  }
  return a.type == cudaMemoryTypeHost ? a.devicePointer : nullptr;
}

extern "C" se2m_status se2m_query(se2m_map* m, int64_t n, const double* xyt, float* risk, float* pitch, float* roll,
                                  float* z, uint8_t* trav) {
  SE2M_ENTER(m);
  if (n < 0 || (n > 0 && !xyt) || n > (1ll << 30)) return fail(m, SE2M_ERR_INVALID_ARG, "query: bad n / xyt");
  if (n == 0) return SE2M_OK;
  se2m_status st = stage_queries(m, n, xyt);
  if (st != SE2M_OK) return st;
  AssessParams p = make_params(m);
  CUDA_TRY(m, launch_query(p, query_geo(m), (int)n, m->d_qxyt, m->d_qout, m->d_qcnt, m->stream), "query kernel");
  m->launches++;
  std::vector<float> out((size_t)n * 5);
  int n_out = 0;
  CUDA_TRY(m, cudaMemcpyAsync(out.data(), m->d_qout, out.size() * sizeof(float), cudaMemcpyDeviceToHost, m->stream), "D2H query");
  CUDA_TRY(m, cudaMemcpyAsync(&n_out, m->d_qcnt, sizeof(int), cudaMemcpyDeviceToHost, m->stream), "D2H query");
  CUDA_TRY(m, cudaStreamSynchronize(m->stream), "sync(query)");
  if (risk) memcpy(risk, out.data(), n * sizeof(float));
  if (pitch) memcpy(pitch, out.data() + n, n * sizeof(float));
  if (roll) memcpy(roll, out.data() + 2 * n, n * sizeof(float));
  if (z) memcpy(z, out.data() + 3 * n, n * sizeof(float));
  if (trav)
    for (int64_t q = 0; q < n; ++q) trav[q] = out[4 * n + q] > 0.5f ? 1 : 0;
  return n_out ? fail(m, SE2M_ERR_OUT_OF_RANGE, "query: some states outside the window / not owned") : SE2M_OK;
}

extern "C" se2m_status se2m_query_async(se2m_map* m, int64_t n, const double* xyt, float* out, int32_t mem) {
  SE2M_ENTER(m);
  if (n < 0 || (n > 0 && (!xyt || !out)) || n > (1ll << 30) || (mem != SE2M_MEM_HOST && mem != SE2M_MEM_DEVICE))
    return fail(m, SE2M_ERR_INVALID_ARG, "query_async: bad n / pointers / mem");
  if (n == 0) return SE2M_OK;
  AssessParams p = make_params(m);
  void* zx = mem == SE2M_MEM_HOST ? mapped_host(xyt) : nullptr;
  void* zo = zx ? mapped_host(out) : nullptr;
  if (zx && zo) {  // pinned host buffers: the kernel reads and writes them in place
    // (the miss counter is not reported by the async form: no reset on the stream)
    if (!m->d_qcnt) CUDA_TRY(m, cudaMalloc(&m->d_qcnt, sizeof(int)), "cudaMalloc(query)");
    CUDA_TRY(m, launch_query(p, query_geo(m), (int)n, static_cast<const double*>(zx), static_cast<float*>(zo), m->d_qcnt,
                             m->stream), "query kernel");
    m->launches++;
    return SE2M_OK;
  }
  se2m_status st = stage_queries(m, n, xyt);
  if (st != SE2M_OK) return st;
  float* dst = mem == SE2M_MEM_DEVICE ? out : m->d_qout;
  CUDA_TRY(m, launch_query(p, query_geo(m), (int)n, m->d_qxyt, dst, m->d_qcnt, m->stream), "query kernel");
  m->launches++;
  if (mem == SE2M_MEM_HOST)
    CUDA_TRY(m, cudaMemcpyAsync(out, m->d_qout, (size_t)n * 5 * sizeof(float), cudaMemcpyDeviceToHost, m->stream),
             "D2H query");
  return SE2M_OK;
}

extern "C" se2m_status se2m_download(se2m_map* m, float* risk, float* pitch, float* roll, float* z, uint8_t* trav,
                                     int32_t mem) {
  SE2M_ENTER(m);
  if (mem != SE2M_MEM_HOST && mem != SE2M_MEM_DEVICE) return fail(m, SE2M_ERR_INVALID_ARG, "download: bad mem");
  const size_t nst = (size_t)m->prm.nx * m->prm.ny * m->prm.n_yaw;
  AssessParams p = make_params(m);
  const int klo = m->k_lo, khi = m->k_hi;
  // owned bins in full-bin numbering: [klo, khi) and, if paired, [klo+H, khi+H); pass a predicate via the range
  // by gathering twice when paired (the kernel tests k in [k_lo, k_hi)).
  struct Plane { void* dst; int which; size_t esz; } planes[] = {
      {risk, 0, 4}, {pitch, 1, 4}, {roll, 2, 4}, {z, 3, 4}, {trav, 4, 1}};
  for (auto& pl : planes) {
    if (!pl.dst) continue;
    void* target = pl.dst;
    if (mem == SE2M_MEM_HOST) {
      se2m_status st = ensure_stage(m, nst * pl.esz);
      if (st != SE2M_OK) return st;
      target = m->d_stage;
    }
    float* f[4] = {nullptr, nullptr, nullptr, nullptr};
    uint8_t* t = nullptr;
    if (pl.which < 4) f[pl.which] = (float*)target; else t = (uint8_t*)target;
    // pass 1: bins [0, H) owned range; pass 2 (paired): bins [H, 2H)
    if (!m->paired) {
      CUDA_TRY(m, launch_gather_logical(p, klo, khi, f[0], f[1], f[2], f[3], t, m->stream), "gather");
      m->launches++;
    } else {
      // a bin k is owned iff k in [klo, khi) or k in [klo+H, khi+H): one launch with a widened range is
      // only correct for the unsharded case; otherwise gather twice into the same target (second
      // pass overwrites only... ) -> do it with two windows of the same kernel.
      if (klo == 0 && khi == m->H) {
        CUDA_TRY(m, launch_gather_logical(p, 0, m->prm.n_yaw, f[0], f[1], f[2], f[3], t, m->stream), "gather");
        m->launches++;
      } else {
        AssessParams q1 = p;
        q1.n_yaw = m->H;  // bins [0, H)
        CUDA_TRY(m, launch_gather_logical(q1, klo, khi, f[0], f[1], f[2], f[3], t, m->stream), "gather");
        AssessParams q2 = p;
        const size_t plane = (size_t)m->prm.nx * m->prm.ny;
        q2.n_yaw = m->H;
        q2.out += plane * m->H;
        q2.trav += (size_t)m->H * m->prm.ny * m->trav_words;
        float* g[4];
        for (int i = 0; i < 4; ++i) g[i] = f[i] ? f[i] + plane * m->H : nullptr;
        CUDA_TRY(m, launch_gather_logical(q2, klo, khi, g[0], g[1], g[2], g[3], t ? t + plane * m->H : nullptr, m->stream), "gather");
        m->launches += 2;
      }
    }
    if (mem == SE2M_MEM_HOST)
      CUDA_TRY(m, cudaMemcpyAsync(pl.dst, m->d_stage, nst * pl.esz, cudaMemcpyDeviceToHost, m->stream), "D2H download");
  }
  CUDA_TRY(m, cudaStreamSynchronize(m->stream), "sync(download)");
  return SE2M_OK;
}

extern "C" se2m_status se2m_download_compact(se2m_map* m, uint16_t* risk_h, uint32_t* trav_bits, int32_t mem) {
  SE2M_ENTER(m);
  if (mem != SE2M_MEM_HOST && mem != SE2M_MEM_DEVICE) return fail(m, SE2M_ERR_INVALID_ARG, "download_compact: bad mem");
  const int wpr = (m->prm.nx + 31) / 32;
  const size_t nst = (size_t)m->prm.nx * m->prm.ny * m->prm.n_yaw;
  const size_t rb = risk_h ? nst * 2 : 0, bb = trav_bits ? (size_t)m->prm.n_yaw * m->prm.ny * wpr * 4 : 0;
  if (!rb && !bb) return SE2M_OK;
  uint16_t* dr = risk_h;
  uint32_t* db = trav_bits;
  if (mem == SE2M_MEM_HOST) {
    se2m_status st = ensure_stage(m, rb + bb);
    if (st != SE2M_OK) return st;
    dr = risk_h ? reinterpret_cast<uint16_t*>(m->d_stage) : nullptr;
    db = trav_bits ? reinterpret_cast<uint32_t*>(reinterpret_cast<char*>(m->d_stage) + rb) : nullptr;
  }
  AssessParams p = make_params(m);
  // owned full bins: [k_lo, k_hi) and, if paired, [k_lo + H, k_hi + H) -> two launches over half planes
  if (!m->paired || (m->k_lo == 0 && m->k_hi == m->H)) {
    CUDA_TRY(m, launch_gather_compact(p, m->paired ? 0 : m->k_lo, m->paired ? m->prm.n_yaw : m->k_hi, dr, db, wpr,
                                      m->stream), "gather_compact");
    m->launches++;
  } else {
    const size_t plane = (size_t)m->prm.nx * m->prm.ny;
    for (int half = 0; half < 2; ++half) {
      AssessParams q = p;
      q.n_yaw = m->H;
      q.out += plane * m->H * half;
      q.trav += (size_t)m->H * m->prm.ny * m->trav_words * half;
      CUDA_TRY(m, launch_gather_compact(q, m->k_lo, m->k_hi, dr ? dr + plane * m->H * half : nullptr,
                                        db ? db + (size_t)m->H * m->prm.ny * wpr * half : nullptr, wpr, m->stream),
               "gather_compact");
      m->launches++;
    }
  }
  if (mem == SE2M_MEM_HOST) {
    if (risk_h) CUDA_TRY(m, cudaMemcpyAsync(risk_h, dr, rb, cudaMemcpyDeviceToHost, m->stream), "D2H risk_h");
    if (trav_bits) CUDA_TRY(m, cudaMemcpyAsync(trav_bits, db, bb, cudaMemcpyDeviceToHost, m->stream), "D2H bits");
  }
  CUDA_TRY(m, cudaStreamSynchronize(m->stream), "sync(download_compact)");
  return SE2M_OK;
}

// logical rows of the window this rank owns under row-band sharding (all rows otherwise)
static int owned_rows(const se2m_map* m, int32_t* rows) {
  const bool sh = m->prm.shard_mode == SE2M_SHARD_ROWS && m->prm.world_size > 1;
  const int TY = tile_rows(m->R_T), G = m->prm.world_size;
  int n = 0;
  for (int j = 0; j < m->prm.ny; ++j) {
    const long long J = m->J_M + j;
    if (!sh || pmod(floor_div(J, TY) - m->prm.rank, G) == 0) {
      if (rows) rows[n] = j;
      ++n;
    }
  }
  return n;
}

extern "C" se2m_status se2m_owned_rows(const se2m_map* m, int32_t* rows, int32_t* n) {
  if (!m || !n) return SE2M_ERR_INVALID_ARG;
  *n = owned_rows(m, rows);
  return SE2M_OK;
}

extern "C" se2m_status se2m_download_compact_rep(se2m_map* m, uint16_t* risk_h, uint32_t* trav_bits, int32_t mem) {
  SE2M_ENTER(m);
  if (mem != SE2M_MEM_HOST && mem != SE2M_MEM_DEVICE) return fail(m, SE2M_ERR_INVALID_ARG, "download_compact_rep: bad mem");
  const int wpr = (m->prm.nx + 31) / 32;
  const int n_rep = m->paired ? m->H : m->prm.n_yaw;
  // row-band sharding: only the rank's own rows, packed (se2m_owned_rows lists them)
  const bool packed = m->prm.shard_mode == SE2M_SHARD_ROWS && m->prm.world_size > 1;
  const int rows = packed ? owned_rows(m, nullptr) : m->prm.ny;
  const size_t plane = (size_t)m->prm.nx * rows;
  const size_t rb = risk_h ? plane * n_rep * 2 : 0, bb = trav_bits ? (size_t)n_rep * rows * wpr * 4 : 0;
  if (!rb && !bb) return SE2M_OK;
  AssessParams p = make_params(m);
  p.n_yaw = n_rep;  // planes [0, n_rep): the representative bins (or all bins when n_yaw is odd)
  const int klo = m->k_lo, khi = m->k_hi;  // owned representative bins (others: risk 1.0 / trav 0)
  if (mem == SE2M_MEM_DEVICE) {
    CUDA_TRY(m, launch_gather_compact(p, klo, khi, risk_h, trav_bits, wpr, m->stream, packed ? rows : 0),
             "gather_compact");
    m->launches++;
    return SE2M_OK;
  }
  if (!m->copy_stream) {
    CUDA_TRY(m, cudaStreamCreateWithFlags(&m->copy_stream, cudaStreamNonBlocking), "cudaStreamCreate(copy)");
    for (int b = 0; b < 2; ++b) {
      CUDA_TRY(m, cudaEventCreateWithFlags(&m->ev_gathered[b], cudaEventDisableTiming), "cudaEventCreate");
      CUDA_TRY(m, cudaEventCreateWithFlags(&m->ev_copied[b], cudaEventDisableTiming), "cudaEventCreate");
    }
  }
  if (m->rep_bytes < rb + bb) {
    CUDA_TRY(m, cudaStreamSynchronize(m->copy_stream), "sync(copy stream)");
    CUDA_TRY(m, cudaStreamSynchronize(m->stream), "sync");
    for (int b = 0; b < 2; ++b) {
      if (m->d_rep[b]) cudaFree(m->d_rep[b]);
      m->d_rep[b] = nullptr;
    }
    m->rep_bytes = 0;
    for (int b = 0; b < 2; ++b) CUDA_TRY(m, cudaMalloc(&m->d_rep[b], rb + bb), "cudaMalloc(rep staging)");
    m->rep_bytes = rb + bb;
  }
  const int b = m->rep_slot;
  m->rep_slot ^= 1;
  uint16_t* dr = risk_h ? reinterpret_cast<uint16_t*>(m->d_rep[b]) : nullptr;
  uint32_t* db = trav_bits ? reinterpret_cast<uint32_t*>(m->d_rep[b] + rb) : nullptr;
  // staging b is reused only after its previous D2H finished; the D2H waits for the gather
  CUDA_TRY(m, cudaStreamWaitEvent(m->stream, m->ev_copied[b], 0), "wait(copied)");
  CUDA_TRY(m, launch_gather_compact(p, klo, khi, dr, db, wpr, m->stream, packed ? rows : 0), "gather_compact");
  m->launches++;
  CUDA_TRY(m, cudaEventRecord(m->ev_gathered[b], m->stream), "record(gathered)");
  CUDA_TRY(m, cudaStreamWaitEvent(m->copy_stream, m->ev_gathered[b], 0), "wait(gathered)");
  if (risk_h) CUDA_TRY(m, cudaMemcpyAsync(risk_h, dr, rb, cudaMemcpyDeviceToHost, m->copy_stream), "D2H risk_h");
  if (trav_bits) CUDA_TRY(m, cudaMemcpyAsync(trav_bits, db, bb, cudaMemcpyDeviceToHost, m->copy_stream), "D2H bits");
  CUDA_TRY(m, cudaEventRecord(m->ev_copied[b], m->copy_stream), "record(copied)");
  return SE2M_OK;
}

// ---- NEXT-1: LiDAR frame integration --------------------------------------------------------------------
extern "C" se2m_status se2m_integrate_scan(se2m_map* m, const float* points, int64_t n, const se2m_pose* pose,
                                           int32_t mem, int64_t* out_counts) {
  SE2M_ENTER(m);
  if (n < 0 || n > (1ll << 30) || (n > 0 && !points) || !pose || (mem != SE2M_MEM_HOST && mem != SE2M_MEM_DEVICE))
    return fail(m, SE2M_ERR_INVALID_ARG, "integrate_scan: bad arguments");
  if (out_counts) memset(out_counts, 0, 5 * sizeof(int64_t));
  if (n == 0) return SE2M_OK;
  FrontendScratch& s = m->fe;
  if ((size_t)n > s.cap) {
    cudaStreamSynchronize(m->stream);
    void* old[] = {s.key, s.idx, s.skey, s.sidx, s.meas, s.temp, m->d_pts};
    for (void* q : old) if (q) cudaFree(q);
    s.key = s.idx = s.skey = s.sidx = nullptr; s.meas = nullptr; s.temp = nullptr; m->d_pts = nullptr;
    s.cap = 0;
    s.temp_bytes = frontend_temp_bytes((int)n);
    CUDA_TRY(m, cudaMalloc(&s.key, n * sizeof(int)), "cudaMalloc(fe)");
    CUDA_TRY(m, cudaMalloc(&s.idx, n * sizeof(int)), "cudaMalloc(fe)");
    CUDA_TRY(m, cudaMalloc(&s.skey, n * sizeof(int)), "cudaMalloc(fe)");
    CUDA_TRY(m, cudaMalloc(&s.sidx, n * sizeof(int)), "cudaMalloc(fe)");
    CUDA_TRY(m, cudaMalloc(&s.meas, n * sizeof(double4)), "cudaMalloc(fe)");
    CUDA_TRY(m, cudaMalloc(&s.temp, std::max<size_t>(s.temp_bytes, 16)), "cudaMalloc(fe)");
    CUDA_TRY(m, cudaMalloc(&m->d_pts, n * 3 * sizeof(float)), "cudaMalloc(fe)");
    s.cap = (size_t)n;
  }
  if (!s.counts) CUDA_TRY(m, cudaMalloc(&s.counts, 5 * sizeof(int)), "cudaMalloc(fe)");
  if (!s.bbox) CUDA_TRY(m, cudaMalloc(&s.bbox, 4 * sizeof(int)), "cudaMalloc(fe)");
  const float* pts = points;
  if (mem == SE2M_MEM_HOST) {
    CUDA_TRY(m, cudaMemcpyAsync(m->d_pts, points, n * 3 * sizeof(float), cudaMemcpyHostToDevice, m->stream), "H2D points");
    pts = m->d_pts;
  }
  const int bbox0[4] = {INT32_MAX, -1, INT32_MAX, -1};
  CUDA_TRY(m, cudaMemsetAsync(s.counts, 0, 5 * sizeof(int), m->stream), "fe counts");
  CUDA_TRY(m, cudaMemcpyAsync(s.bbox, bbox0, sizeof bbox0, cudaMemcpyHostToDevice, m->stream), "fe bbox");
  FrontendArgs a;
  memset(&a, 0, sizeof a);
  memcpy(a.pose.R_B, pose->R_B, sizeof a.pose.R_B); memcpy(a.pose.p_B, pose->p_B, sizeof a.pose.p_B);
  memcpy(a.pose.R_BS, pose->R_BS, sizeof a.pose.R_BS); memcpy(a.pose.p_BS, pose->p_BS, sizeof a.pose.p_BS);
  memcpy(a.pose.Sigma_S, pose->Sigma_S, sizeof a.pose.Sigma_S);
  memcpy(a.pose.Sigma_R, pose->Sigma_R, sizeof a.pose.Sigma_R);
  memcpy(a.pose.Sigma_B, pose->Sigma_B, sizeof a.pose.Sigma_B);
  a.r = m->prm.resolution; a.z_min = m->prm.fe_z_min; a.z_max = m->prm.fe_z_max;
  a.gate = m->prm.fe_gate; a.ray_eps = m->prm.fe_ray_eps;
  const double* RB = pose->R_B;
  const double* pbs = pose->p_BS;
  a.sx = (RB[0] * pbs[0] + RB[1] * pbs[1] + RB[2] * pbs[2]) + pose->p_B[0];  // R_B p_BS + p_B, left to right
  a.sy = (RB[3] * pbs[0] + RB[4] * pbs[1] + RB[5] * pbs[2]) + pose->p_B[1];
  a.sz = (RB[6] * pbs[0] + RB[7] * pbs[1] + RB[8] * pbs[2]) + pose->p_B[2];
  a.I_M = m->I_M; a.J_M = m->J_M;
  a.nx = m->prm.nx; a.ny = m->prm.ny; a.ldh = m->ldh;
  a.key_bits = 1;
  while ((1ll << a.key_bits) - 1 <= (long long)m->ldh * m->prm.ny) ++a.key_bits;  // indices < 2^bits - 1
  a.key_none = (int)((1ll << a.key_bits) - 1);
  a.pxM = pmod(m->I_M, m->prm.nx); a.pyM = pmod(m->J_M, m->prm.ny);
  CUDA_TRY(m, frontend_run(a, (int)n, pts, s, m->d_h, m->d_var, m->stream), "front-end kernels");
  m->launches += 3;
  int cnt[5], bb[4];
  CUDA_TRY(m, cudaMemcpyAsync(cnt, s.counts, sizeof cnt, cudaMemcpyDeviceToHost, m->stream), "D2H fe");
  CUDA_TRY(m, cudaMemcpyAsync(bb, s.bbox, sizeof bb, cudaMemcpyDeviceToHost, m->stream), "D2H fe");
  CUDA_TRY(m, cudaStreamSynchronize(m->stream), "sync(fe)");
  if (out_counts)
    for (int i = 0; i < 5; ++i) out_counts[i] = cnt[i];
  if (bb[1] >= 0) {  // touched cells -> dirty (H9)
    m->dirty.push_back(Rect{m->I_M + bb[0], m->I_M + bb[1] + 1, m->J_M + bb[2], m->J_M + bb[3] + 1});
    m->have_data = true;
    m->inpaint_valid = false;
  }
  return SE2M_OK;
}

static se2m_status ring_to_logical(se2m_map* m, const float* ring, float* dst_dev) {
  // the ring (pitch ldh) in logical order (pitch nx): one 2-D copy per quadrant of the seam
  const int nx = m->prm.nx, ny = m->prm.ny, pxM = pmod(m->I_M, nx), pyM = pmod(m->J_M, ny);
  const int xs[2][3] = {{0, pxM, nx - pxM}, {nx - pxM, 0, pxM}};  // (logical x0, physical x0, width)
  const int ys[2][3] = {{0, pyM, ny - pyM}, {ny - pyM, 0, pyM}};
  for (auto& X : xs)
    for (auto& Y : ys)
      if (X[2] > 0 && Y[2] > 0)
        CUDA_TRY(m, cudaMemcpy2DAsync(dst_dev + (size_t)Y[0] * nx + X[0], (size_t)nx * 4,
                                      ring + (size_t)Y[1] * m->ldh + X[1], (size_t)m->ldh * 4, (size_t)X[2] * 4, Y[2],
                                      cudaMemcpyDeviceToDevice, m->stream), "ring gather");
  return SE2M_OK;
}

extern "C" se2m_status se2m_download_elevation(se2m_map* m, float* heights, float* variances, int32_t mem) {
  SE2M_ENTER(m);
  if (mem != SE2M_MEM_HOST && mem != SE2M_MEM_DEVICE) return fail(m, SE2M_ERR_INVALID_ARG, "download_elevation: bad mem");
  const size_t cells = (size_t)m->prm.nx * m->prm.ny;
  const float* rings[2] = {m->d_h, m->d_var};
  float* outs[2] = {heights, variances};
  for (int q = 0; q < 2; ++q) {
    if (!outs[q]) continue;
    float* target = outs[q];
    if (mem == SE2M_MEM_HOST) {
      se2m_status st = ensure_stage(m, cells * 4);
      if (st != SE2M_OK) return st;
      target = m->d_stage;
    }
    se2m_status st = ring_to_logical(m, rings[q], target);
    if (st != SE2M_OK) return st;
    if (mem == SE2M_MEM_HOST)
      CUDA_TRY(m, cudaMemcpyAsync(outs[q], target, cells * 4, cudaMemcpyDeviceToHost, m->stream), "D2H elevation");
    CUDA_TRY(m, cudaStreamSynchronize(m->stream), "sync(download_elevation)");
  }
  return SE2M_OK;
}

extern "C" se2m_status se2m_download_inpainted(se2m_map* m, float* heights, int32_t mem) {
  SE2M_ENTER(m);
  if (!heights || (mem != SE2M_MEM_HOST && mem != SE2M_MEM_DEVICE))
    return fail(m, SE2M_ERR_INVALID_ARG, "download_inpainted: bad pointer / mem");
  if (!m->inpaint_valid) {
    se2m_status st = run_inpaint(m, nullptr);
    if (st != SE2M_OK) return st;
  }
  const size_t bytes = (size_t)m->prm.nx * m->prm.ny * 4;
  if (mem == SE2M_MEM_DEVICE) return ring_to_logical(m, m->d_hin, heights);
  se2m_status st = ensure_stage(m, bytes);
  if (st != SE2M_OK) return st;
  st = ring_to_logical(m, m->d_hin, m->d_stage);
  if (st != SE2M_OK) return st;
  CUDA_TRY(m, cudaMemcpyAsync(heights, m->d_stage, bytes, cudaMemcpyDeviceToHost, m->stream), "D2H inpainted");
  CUDA_TRY(m, cudaStreamSynchronize(m->stream), "sync");
  return SE2M_OK;
}

// ---- NEXT-2: SDF of the explicit-obstacle set --------------------------------------------------------
static int sdf_radius(double d_max, double r) { return (int)ceil(d_max / r - 1e-9); }

extern "C" se2m_status se2m_compute_sdf(se2m_map* m, double d_max) {
  SE2M_ENTER(m);
  if (!(d_max > 0) || !isfinite(d_max)) return fail(m, SE2M_ERR_INVALID_ARG, "compute_sdf: d_max must be > 0");
  const int W = sdf_radius(d_max, m->prm.resolution);
  if (W > 96) return fail(m, SE2M_ERR_UNSUPPORTED, "compute_sdf: d_max / resolution > 96 cells");
  if (m->prm.shard_mode == SE2M_SHARD_ROWS && m->prm.world_size > 1)
    return fail(m, SE2M_ERR_UNSUPPORTED, "compute_sdf: needs whole layers (not available with row sharding)");
  if (!m->have_data) return fail(m, SE2M_ERR_STATE, "compute_sdf before any assess");
  // the obstacle set is the last assess's: stale once the window moved or cells changed since then
  if (m->all_dirty || !m->dirty.empty() || (m->prm.inpaint && !m->inpaint_valid))
    return fail(m, SE2M_ERR_STATE, "compute_sdf: the risk map is stale (assess after the last shift / update)");
  const size_t plane = (size_t)m->prm.nx * m->prm.ny;
  if (!m->d_sdf) {
    CUDA_TRY(m, cudaMalloc(&m->d_sdf, plane * m->H * sizeof(float)), "cudaMalloc(sdf)");
    // layers of representative bins this rank does not own (yaw shards) stay NaN (never written)
    CUDA_TRY(m, cudaMemsetAsync(m->d_sdf, 0xff, plane * m->H * sizeof(float), m->stream), "sdf init");
  }
  if (!m->d_sdf_g) CUDA_TRY(m, cudaMalloc(&m->d_sdf_g, plane * m->H * sizeof(uint16_t)), "cudaMalloc(sdf scratch)");
  SdfParams sp;
  memset(&sp, 0, sizeof sp);
  sp.nx = m->prm.nx; sp.ny = m->prm.ny; sp.layers = m->k_hi - m->k_lo;
  sp.r = (float)m->prm.resolution; sp.d_max = (float)d_max; sp.W = W;
  sp.trav = m->d_trav + (size_t)m->k_lo * m->prm.ny * m->trav_words;
  sp.trav_words = m->trav_words; sp.pxM = pmod(m->I_M, m->prm.nx); sp.pyM = pmod(m->J_M, m->prm.ny);
  sp.I_M = m->I_M;
  sp.out = m->d_sdf + plane * m->k_lo;
  sp.g = m->d_sdf_g;
  CUDA_TRY(m, launch_sdf(sp, m->stream), "sdf kernels");
  m->launches += 2;
  m->sdf_valid = true;
  m->sdf_dmax = d_max;
  return SE2M_OK;
}

extern "C" se2m_status se2m_sdf_from_mask(const uint8_t* mask, int32_t nx, int32_t ny, int32_t layers,
                                          double resolution, double d_max, float* out, int32_t mem,
                                          int32_t device) {
  if (!mask || !out || nx < 1 || ny < 1 || layers < 1 || !(resolution > 0) || !(d_max > 0) ||
      (mem != SE2M_MEM_HOST && mem != SE2M_MEM_DEVICE))
    return fail(nullptr, SE2M_ERR_INVALID_ARG, "sdf_from_mask: bad arguments");
  const int W = sdf_radius(d_max, resolution);
  if (W > 96) return fail(nullptr, SE2M_ERR_UNSUPPORTED, "sdf_from_mask: d_max / resolution > 96 cells");
  int n_dev = 0;
  cudaError_t e = cudaGetDeviceCount(&n_dev);
  if (e != cudaSuccess) return fail(nullptr, SE2M_ERR_CUDA, cudaGetErrorString(e));
  if (device < 0 || device >= n_dev) return fail(nullptr, SE2M_ERR_INVALID_ARG, "sdf_from_mask: device ordinal out of range");
  DevGuard dev_guard_(device);
  const size_t n = (size_t)nx * ny * layers;
  uint8_t* dm = const_cast<uint8_t*>(mask);
  float* dout = out;
  if (mem == SE2M_MEM_HOST) {
    if ((e = cudaMalloc(&dm, n)) != cudaSuccess) return fail(nullptr, SE2M_ERR_OOM, "cudaMalloc(mask)");
    if ((e = cudaMalloc(&dout, n * 4)) != cudaSuccess) { cudaFree(dm); return fail(nullptr, SE2M_ERR_OOM, "cudaMalloc(sdf)"); }
    e = cudaMemcpy(dm, mask, n, cudaMemcpyHostToDevice);
  }
  SdfParams sp;
  memset(&sp, 0, sizeof sp);
  sp.nx = nx; sp.ny = ny; sp.layers = layers; sp.r = (float)resolution; sp.d_max = (float)d_max; sp.W = W;
  sp.mask = dm; sp.out = dout;
  uint16_t* dg = nullptr;
  if (e == cudaSuccess && cudaMalloc(&dg, n * sizeof(uint16_t)) != cudaSuccess) {
    if (mem == SE2M_MEM_HOST) { cudaFree(dm); cudaFree(dout); }
    return fail(nullptr, SE2M_ERR_OOM, "cudaMalloc(sdf scratch)");
  }
  sp.g = dg;
  if (e == cudaSuccess) e = launch_sdf(sp, 0);
  if (e == cudaSuccess) e = cudaDeviceSynchronize();
  if (e == cudaSuccess && mem == SE2M_MEM_HOST) e = cudaMemcpy(out, dout, n * 4, cudaMemcpyDeviceToHost);
  cudaFree(dg);
  if (mem == SE2M_MEM_HOST) { cudaFree(dm); cudaFree(dout); }
  return e == cudaSuccess ? SE2M_OK : fail(nullptr, SE2M_ERR_CUDA, cudaGetErrorString(e));
}

// ---- NEXT-3: trilinear query of Risk / SDF with gradient ------------------------------
extern "C" se2m_status se2m_query_trilinear(se2m_map* m, int64_t n, const double* xyt, int32_t field,
                                            float* value, float* grad) {
  SE2M_ENTER(m);
  if (n < 0 || (n > 0 && !xyt) || n > (1ll << 30) || (field != 0 && field != 1))
    return fail(m, SE2M_ERR_INVALID_ARG, "query_trilinear: bad n / xyt / field");
  if (field == 1 && !m->sdf_valid) return fail(m, SE2M_ERR_STATE, "query_trilinear: no SDF (call se2m_compute_sdf)");
  if (n == 0) return SE2M_OK;
  se2m_status st = stage_queries(m, n, xyt);
  if (st != SE2M_OK) return st;
  const float* f = field == 0 ? reinterpret_cast<const float*>(m->d_out) : m->d_sdf;
  CUDA_TRY(m, launch_trilinear(f, field == 0 ? 4 : 1, field, query_geo(m), (int)n, m->d_qxyt, m->d_qout, m->d_qcnt,
                               m->stream), "trilinear kernel");
  m->launches++;
  std::vector<float> out((size_t)n * 4);
  int n_out = 0;
  CUDA_TRY(m, cudaMemcpyAsync(out.data(), m->d_qout, out.size() * sizeof(float), cudaMemcpyDeviceToHost, m->stream),
           "D2H trilinear");
  CUDA_TRY(m, cudaMemcpyAsync(&n_out, m->d_qcnt, sizeof(int), cudaMemcpyDeviceToHost, m->stream), "D2H trilinear");
  CUDA_TRY(m, cudaStreamSynchronize(m->stream), "sync(trilinear)");
  if (value) memcpy(value, out.data(), n * sizeof(float));
  if (grad)
    for (int64_t t = 0; t < n; ++t) {
      grad[3 * t] = out[n + t]; grad[3 * t + 1] = out[2 * n + t]; grad[3 * t + 2] = out[3 * n + t];
    }
  return n_out ? fail(m, SE2M_ERR_OUT_OF_RANGE, "query_trilinear: some corners outside the window / not owned")
               : SE2M_OK;
}

extern "C" se2m_status se2m_query_trilinear_async(se2m_map* m, int64_t n, const double* xyt, int32_t field, float* out,
                                                  int32_t mem) {
  SE2M_ENTER(m);
  if (n < 0 || (n > 0 && (!xyt || !out)) || n > (1ll << 30) || (field != 0 && field != 1) ||
      (mem != SE2M_MEM_HOST && mem != SE2M_MEM_DEVICE))
    return fail(m, SE2M_ERR_INVALID_ARG, "query_trilinear_async: bad n / pointers / field / mem");
  if (field == 1 && !m->sdf_valid) return fail(m, SE2M_ERR_STATE, "query_trilinear_async: no SDF (call se2m_compute_sdf)");
  if (n == 0) return SE2M_OK;
  const float* f = field == 0 ? reinterpret_cast<const float*>(m->d_out) : m->d_sdf;
  void* zx = mem == SE2M_MEM_HOST ? mapped_host(xyt) : nullptr;
  void* zo = zx ? mapped_host(out) : nullptr;
  if (zx && zo) {  // pinned host buffers: read and written in place by the kernel (miss counter not reported)
    if (!m->d_qcnt) CUDA_TRY(m, cudaMalloc(&m->d_qcnt, sizeof(int)), "cudaMalloc(query)");
    CUDA_TRY(m, launch_trilinear(f, field == 0 ? 4 : 1, field, query_geo(m), (int)n, static_cast<const double*>(zx),
                                 static_cast<float*>(zo), m->d_qcnt, m->stream), "trilinear kernel");
    m->launches++;
    return SE2M_OK;
  }
  se2m_status st = stage_queries(m, n, xyt);
  if (st != SE2M_OK) return st;
  float* dst = mem == SE2M_MEM_DEVICE ? out : m->d_qout;
  CUDA_TRY(m, launch_trilinear(f, field == 0 ? 4 : 1, field, query_geo(m), (int)n, m->d_qxyt, dst, m->d_qcnt, m->stream),
           "trilinear kernel");
  m->launches++;
  if (mem == SE2M_MEM_HOST)
    CUDA_TRY(m, cudaMemcpyAsync(out, m->d_qout, (size_t)n * 4 * sizeof(float), cudaMemcpyDeviceToHost, m->stream),
             "D2H trilinear");
  return SE2M_OK;
}

// SDF planes in logical order: out[k][j][i] for all n_yaw bins (bins k and k + n/2 share a layer).
extern "C" se2m_status se2m_download_sdf(se2m_map* m, float* out, int32_t mem) {
  SE2M_ENTER(m);
  if (!out || (mem != SE2M_MEM_HOST && mem != SE2M_MEM_DEVICE)) return fail(m, SE2M_ERR_INVALID_ARG, "download_sdf: bad pointer / mem");
  if (!m->sdf_valid) return fail(m, SE2M_ERR_STATE, "download_sdf: no SDF (call se2m_compute_sdf)");
  const int nx = m->prm.nx, ny = m->prm.ny;
  const size_t plane = (size_t)nx * ny, nst = plane * m->prm.n_yaw;
  float* target = out;
  if (mem == SE2M_MEM_HOST) {
    se2m_status st = ensure_stage(m, nst * 4);
    if (st != SE2M_OK) return st;
    target = m->d_stage;
  }
  // one 2-D strided copy per logical quadrant of the ring (no extra kernel): rows [0, ny - pyM) come from
  // physical rows [pyM, ny), the rest from [0, pyM); same split in x
  const int pxM = pmod(m->I_M, nx), pyM = pmod(m->J_M, ny);
  for (int k = 0; k < m->prm.n_yaw; ++k) {
    const int L = m->paired ? k % m->H : k;
    const float* src = m->d_sdf + plane * L;
    float* dst = target + plane * k;
    const int xs[2][3] = {{0, pxM, nx - pxM}, {nx - pxM, 0, pxM}};  // (logical x0, physical x0, width)
    const int ys[2][3] = {{0, pyM, ny - pyM}, {ny - pyM, 0, pyM}};
    for (auto& X : xs)
      for (auto& Y : ys)
        if (X[2] > 0 && Y[2] > 0)
          CUDA_TRY(m, cudaMemcpy2DAsync(dst + (size_t)Y[0] * nx + X[0], (size_t)nx * 4, src + (size_t)Y[1] * nx + X[1],
                                        (size_t)nx * 4, (size_t)X[2] * 4, Y[2], cudaMemcpyDeviceToDevice, m->stream),
                   "sdf gather");
  }
  if (mem == SE2M_MEM_HOST)
    CUDA_TRY(m, cudaMemcpyAsync(out, target, nst * 4, cudaMemcpyDeviceToHost, m->stream), "D2H sdf");
  CUDA_TRY(m, cudaStreamSynchronize(m->stream), "sync(download_sdf)");
  return SE2M_OK;
}

extern "C" se2m_status se2m_get_origin(const se2m_map* m, int64_t* I_M, int64_t* J_M) {
  if (!m) return SE2M_ERR_INVALID_ARG;
  if (I_M) *I_M = m->I_M;
  if (J_M) *J_M = m->J_M;
  return SE2M_OK;
}

extern "C" se2m_status se2m_stencil_info(const se2m_map* m, int32_t k, int32_t* n_cells, int32_t* radius) {
  if (!m || k < 0 || k >= m->prm.n_yaw) return SE2M_ERR_INVALID_ARG;
  const int kr = (m->paired && k >= m->H) ? k - m->H : k;
  if (n_cells) *n_cells = m->ncells[kr];
  if (radius) *radius = m->R;
  return SE2M_OK;
}

extern "C" se2m_status se2m_synchronize(se2m_map* m) {
  SE2M_ENTER(m);
  CUDA_TRY(m, cudaStreamSynchronize(m->stream), "synchronize");
  if (m->copy_stream) CUDA_TRY(m, cudaStreamSynchronize(m->copy_stream), "synchronize(copy stream)");
  return SE2M_OK;
}

extern "C" int64_t se2m_launch_count(const se2m_map* m) { return m ? m->launches : 0; }

extern "C" se2m_status se2m_debug_phases(se2m_map* m, void* out, int64_t max_records, int32_t reset, int64_t* n) {
  SE2M_ENTER(m);
  long long cnt = 0;
  const cudaError_t e = debug_phases(out, max_records, reset, &cnt, m->stream);
  if (n) *n = cnt;
  if (e == cudaErrorNotSupported) return fail(m, SE2M_ERR_UNSUPPORTED, "debug_phases: library built without SE2M_PHASES");
  if (e != cudaSuccess) return cuda_fail(m, e, "debug_phases");
  return SE2M_OK;
}

extern "C" const char* se2m_last_error(const se2m_map* m) {
  return m ? m->err.c_str() : g_init_error.c_str();
}
