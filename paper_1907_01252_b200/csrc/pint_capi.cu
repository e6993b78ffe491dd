// Host runtime of the batched fine propagator: context (mesh tables, multigrid
// hierarchy, Krylov / Newton workspace), the Newton + GMRES + V-cycle control
// flow, and the C ABI declared in include/pint_b200.h.
//
// Control flow mirrors the reference hot path (SURVEY.md §3 stack A):
//   ThetaPropagator.advance (integrators.py:144-166)   -> pint_propagate
//   _theta_step (integrators.py:70-96)                  -> Impl::newton_step
//   newton_solve (linalg.py:167-248)                    -> Impl::newton_step
//   _fd_jacobian + np.linalg.solve (linalg.py:152-164, 224)
//                      -> Jacobian assembly + V-cycle-preconditioned GMRES
// Every slice carries its own Newton / line-search / Krylov state; kernels
// skip inactive slices, so a slice's arithmetic is independent of the batch.
#include <cuda_runtime.h>

#include <algorithm>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <functional>
#include <map>
#include <mutex>
#include <set>
#include <tuple>
#include <utility>
#include <string>
#include <vector>

#include "../../include/pint_b200.h"
#include "kernels_assembly.cuh"
#include "kernels_linalg.cuh"
#include "kernels_loop.cuh"
#include "kernels_parareal.cuh"

using namespace pint;

namespace {

constexpr int kDenseMax = 1024;
constexpr size_t kTailSmemMax = 220 * 1024;  // dynamic shared memory of a staged tail CTA
constexpr int kCapDepth = 8;      // nesting depth of conditional graph bodies (one capture stream each)
constexpr int kMaxBodies = 16384; // conditional bodies over all loop graphs of a context

struct Level {
  Grid g;
  double* A = nullptr;     // [S][noff][C][C][np]
  double* Dinv = nullptr;  // [S][C][C][np]
  double* rhs = nullptr;
  double* xa = nullptr;
  double* xb = nullptr;
  double* res = nullptr;
  double* sol = nullptr;   // coarse-level V-cycle output (l > 0)
  float* A32 = nullptr;    // fp32 copy of A for the V-cycle's residuals (preconditioner only; level 0 and
                           // the standalone coarse levels above the fused tail)
  float* vinv = nullptr;   // Vanka cell inverses [S][L*L][ncell], fp32 storage (preconditioner only)
  float* vst = nullptr;    // Vanka sweep in block-stencil form [S][noff][C][C][np] (standalone levels; built from vinv)
  double* ycell = nullptr; // Vanka cell corrections [S][L][ncell]
  int ncell = 0;
};

size_t round_up(size_t x, size_t m) { return (x + m - 1) / m * m; }

}  // namespace

struct pint_ctx;
static inline cudaStream_t counted(pint_ctx* ctx, cudaStream_t st);

struct GraphKey {
  int S, j, levels, pre, post, coarse, smoother;
  double omega;
  bool operator<(const GraphKey& o) const {
    return std::tie(S, j, levels, pre, post, coarse, smoother, omega) <
           std::tie(o.S, o.j, o.levels, o.pre, o.post, o.coarse, o.smoother, o.omega);
  }
};

struct pint_ctx {
  pint_problem_desc desc{};
  int D = 2, C = 5, maxS = 0, restart = 30;
  Grid g{};
  Phys ph{};
  int cells[3] = {1, 1, 1};
  std::vector<uint8_t> h_node_flags, h_cell_flags;
  std::vector<double> h_profile;
  uint8_t* d_node_flags = nullptr;
  uint8_t* d_cell_flags = nullptr;
  double* d_profile = nullptr;
  std::vector<Level> lv;
  int dense_n = 0;           // dofs of the coarsest used level (set by precond_setup)
  int dense_cap = 0;         // largest dense dimension the buffer holds
  bool coarse_dense = false; // coarsest used level solved by its dense inverse
  int dense_ld = 0;          // row stride (floats) of the fp32 inverse in d_dense32
  double* d_dense = nullptr;  // fp64 scratch of the single-CTA fallback ([n][2n] augmented)
  float* d_dense32 = nullptr; // coarsest inverse, fp32 [S][n][dense_ld]
  // Newton
  double *ystate = nullptr, *ynew = nullptr, *r = nullptr, *dx = nullptr, *ytrial = nullptr, *rtrial = nullptr,
         *b = nullptr;
  // GMRES
  double *V = nullptr, *H = nullptr, *gv = nullptr, *cs = nullptr, *sn = nullptr, *ybuf = nullptr,
         *w = nullptr, *u = nullptr, *gm_res = nullptr, *gm_tol = nullptr, *gm_beta = nullptr;
  int *gm_active = nullptr, *gm_steps = nullptr, *gm_its = nullptr, *cyc_active = nullptr;
  int* gm_two_pass = nullptr;  // per slice: second Gram-Schmidt pass in this solve
  double* gm_hnorm = nullptr;
  double* Z = nullptr;  // flexible-GMRES preconditioned basis z_j = M^{-1} v_j, [m][S][C][np]
  double* cpart = nullptr;  // fused Arnoldi: CTA partial sums [S][cluster][kMaxBasis]
  unsigned int *ctr_mdot = nullptr, *ctr_norm = nullptr;  // last-block tickets, reset by the last block
  // reductions / per-slice scalars
  double* partial = nullptr;
  int nblk = 0;
  double* d_norms = nullptr;
  int* d_degen = nullptr;
  int* d_active = nullptr;
  int* d_mask2 = nullptr;
  double* d_lam = nullptr;
  StepScalars* d_st = nullptr;
  double* h_dbl = nullptr;  // pinned
  int* h_int = nullptr;     // pinned
  size_t bytes = 0;
  std::vector<void*> allocs;
  std::mutex mu;
  std::string err;
  int prec_levels = 0;  // levels set up by the last precond_setup
  bool use_graphs = true;  // PINT_GRAPHS=0 disables CUDA-graph replay of Arnoldi steps
  std::map<GraphKey, std::pair<cudaGraphExec_t, long long>> graphs;
  cudaStream_t stream = nullptr;  // internal non-blocking stream (capturable)
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  bool verbose = false;  // PINT_VERBOSE=1: per-Newton-iteration trace on stderr
  bool use_tail = true;  // PINT_TAIL=0 disables the fused coarse-level V-cycle kernel
  bool jac_columns = false;  // PINT_JAC=columns: one dual pass per Jacobian column (k_jacobian_colour)
  bool elem_old = false;     // PINT_ELEM=old: per-point K1 / K2' kernels with register gathers (round 1)
  bool vanka_smem = false;   // PINT_VANKA_SETUP=smem: warp-per-cell shared-memory Gauss-Jordan
  int scale_fuse_max = 0;      // PINT_SCALE_FUSE: per-slice length up to which the last norm block scales v_{j+1}
                               // (measured neutral on c1/c2, off)
  int cgs_passes = 0;          // PINT_CGS=1|2 forces the Gram-Schmidt passes per Arnoldi step; 0 = by tolerance
  int cur_passes = 1;          // passes of the running GMRES solve
  bool defer_scale = true;     // PINT_DEFER_SCALE=0: v_{j+1} = w / h by its own launch
  double* defer_w = nullptr;   // set while the V-cycle's first sweep forms v_j from w
  bool host_beta = true;       // PINT_HOST_BETA=0: GMRES recomputes ||b|| on the device (one more sync)
  bool split_norm = false;   // PINT_SPLIT_NORM=1: second CGS update and the norm as two kernels
  bool vanka_split = false;  // PINT_VANKA=split|fused (default split in 3-d): separate k_vanka_cell + k_vanka_gather (y_c buffer)
  std::vector<int> built_step;  // per slice: step of the last multigrid build in this propagate call
  std::vector<int> base_its;    // per slice: Krylov its of the first-Newton-iteration solve after that build
  std::vector<int> first_its;   // per slice: Krylov its of the latest first-Newton-iteration solve
  int poll_every = 4;           // PINT_POLL: Arnoldi steps between host polls of the convergence mask
  bool pdl = true;              // PINT_PDL=0: launch without programmatic stream serialization
  bool jac_strip = true;        // PINT_JAC=colour: 2-d Jacobian by colour-ordered element scatter (k_jacobian_lin)
  bool spmv32_node = true;      // PINT_SPMV32=row: fp32 V-cycle residuals with one thread per (node, row)
  bool spmv32_staged = true;    // PINT_SPMV32=node|row: without the shared-memory staged residual kernel
  int tail_stage = 1;           // PINT_TAIL_STAGE=0: coarsest inverse read from L2 instead of staged in shared memory
  double forcing = 0.5;         // PINT_FORCING: absolute Krylov tolerance of the later Newton iterations / Newton target
                                // (round 1: 0.1; 0.5 keeps Newton at 2.0000 its per step on c2-c4 with 4-7 % fewer Krylov its)
  bool res_strip = false;       // PINT_RES=strip: K1 in node-owner strips (one launch, no zeroing / colour scatter / fix-up;
                                // measured slower: c3 0.64 vs 0.45 ms -- the per-row barriers outweigh the saved passes)
  int res_waves = 4;            // PINT_RES_WAVES: target waves of strip-residual blocks (more chunks, shorter sweeps)
  bool jac_mt = true;           // PINT_JAC_MT=0: one dual pass per direction in the strip Jacobian (round-2 first form)
  bool resid_acc32 = false;     // PINT_RESID_ACC=f32: fp32 accumulation in the staged V-cycle residual
  int strip_w = 25;             // PINT_STRIP_W: owned node columns per Jacobian strip (<= 31)
  bool fuse_prolong = false;    // PINT_FUSE_PROLONG=1: coarse-grid correction inside the post-smoothing residual kernel
                                // (bitwise k_prolong_add + residual; measured slower: c3 863 vs 881, c4 874 vs 879)
  bool vanka_stencil = true;    // PINT_VANKA=fused|split: cell-inverse sweeps instead of the block-stencil form
  size_t spmv32_min = (size_t)2 * 4 * 148 * 128;  // PINT_SPMV32_MIN: nodes x slices from which the staged / node
                                                  // residual kernels replace the (node, row) one
  int tail_rows = 2048;         // PINT_TAIL_ROWS: first level of the fused V-cycle tail has <= this many rows
  int drift_num = 3;            // drift rebuild when 2 its > drift_num base + 4 (PINT_DRIFT; 0 = off)
  int tail_first = -1;   // first level handled by k_vcycle_tail (-1: none)
  int64_t tail_slice_launches = 0;  // profiled tail launches x slices (tail_first == 0)
  bool tail_cluster = true;  // PINT_TAIL_CLUSTER=0: one CTA per slice instead of a cluster
  int tail_cl_force = 0;     // PINT_TAIL_CL=8|4|2: fixed cluster size (else: largest with one wave)
  int num_sms = 148;
  bool use_fused = false;    // PINT_FUSED=1 enables the fused Arnoldi-step kernel (slower than the
                             // graph of level-0 launches on c2: measured 3659 vs 4123 steps*slices/s)
  bool fused = false;        // fused Arnoldi step active for the current hierarchy
  TailArgs tail0{};          // V-cycle description from level 0 (fused path)
  TailArgs tail_cl{};        // the cluster tail's copy (dense rows staged in shared memory)
  unsigned long long* d_work_bytes = nullptr;
  bool fused_used = false;   // profiling: the fused kernel ran while profiling
  TailArgs tail{};
  // profiling (bench.py roofline): launch count and CUDA-event timing of the
  // level-0 smoother sweeps, the dominant kernel of the fine step
  long long launches = 0;
  bool prof = false;
  unsigned long long* d_work = nullptr;  // active-slice launches of the profiled kernel
  std::vector<std::pair<cudaEvent_t, cudaEvent_t>> ev_pairs;
  std::vector<cudaEvent_t> ev_pool;
  size_t ev_used = 0;
  pint_krylov_opts kopt{};
  // matrix-free context (pint_create_ex, PINT_CTX_MATRIX_FREE): no Jacobian,
  // no multigrid hierarchy; GMRES on J(y) w by the K2' kernel, unpreconditioned
  bool matrix_free = false;
  const double* mf_y = nullptr;   // linearisation point of the running matrix-free solve
  const double* mf_yo = nullptr;
  int* gm_cap = nullptr;        // Krylov budget of the running solve (givens_one)
  int* h_cap = nullptr;         // pinned
  // ---- device-driven control flow (Impl::propagate_dev): the whole
  // propagate call as one CUDA graph with conditional WHILE / IF nodes
  bool device_loop = true;      // PINT_DEVICE_LOOP=0: host-driven Newton / GMRES
  int gate = 4;                 // PINT_GATE: Arnoldi steps per conditional IF block
  int gate0 = 12;               // PINT_GATE0: leading Arnoldi steps of a cycle without a gate
  LoopDev ld{};
  LoopScalars* h_ls = nullptr;  // pinned staging of the call scalars
  size_t tab_cap = 0, lsv_cap = 0;
  StepScalars *d_sts = nullptr, *h_sts = nullptr;   // step tables [entries]
  double *d_t1tab = nullptr, *h_t1tab = nullptr;
  int *d_nsteps = nullptr, *h_nsteps = nullptr;
  LoopScalars *d_lsv = nullptr, *h_lsv = nullptr;   // per-slice call scalars of a coarse sweep
  int* h_out_i = nullptr;       // pinned outputs [4][maxS]
  double* h_out_d = nullptr;
  cudaStream_t cap_st[kCapDepth] = {};
  cudaGraph_t cap_root = nullptr;  // root graph of the running capture (conditional handles live here)
  std::set<cudaStream_t> nopdl;    // streams whose next launch must not carry the PDL attribute
  bool capturing = false;          // a loop graph is being captured
  std::map<std::vector<double>, std::pair<cudaGraphExec_t, long long>> loop_graphs;
  std::vector<int> body_nodes;     // kernel nodes per conditional body (host copy)
  int* d_body_nodes = nullptr;
  unsigned long long* d_launch_ctr = nullptr;
  // coarse sweep / boundary-error scratch (grown on demand)
  size_t sw_cap = 0;
  double *sw_part = nullptr, *sw_theta = nullptr, *sw_corr = nullptr, *sw_ft = nullptr;
  int *sw_status = nullptr, *sw_nit = nullptr, *sw_kit = nullptr;
  double* h_sw = nullptr;
  std::vector<void*> grown;  // freed at destroy
};

// CTAs per slice of the V-cycle tail: the largest cluster whose S*CL CTAs run in
// one wave (1: the single-CTA kernel).  Results do not depend on the choice.
static inline int tail_cluster_size(const pint_ctx* ctx, int S) {
  if (!ctx->tail_cluster) return 1;
  if (ctx->tail_cl_force) return ctx->tail_cl_force;
  // measured (profiles/r02_tail_cluster_ab.jsonl): 4 CTAs per slice beat 8 and 2 on c2 (S = 32), c3 (S = 64,
  // two CTAs per SM) and c4 (S = 16); 8 for small batches (c1 S = 10: 7720 vs 6750)
  if (S * 8 <= 96) return 8;  // c1 (S = 10) and the batch-1 coarse sweeps: 8 beats 4 by 14 %
  if (S * 4 <= 2 * ctx->num_sms) return 4;
  if (S * 2 <= 2 * ctx->num_sms) return 2;
  return 1;
}

static inline cudaStream_t counted(pint_ctx* ctx, cudaStream_t st) {
  ++ctx->launches;
  return st;
}

namespace {


// Every kernel launch of the library: counted (profiling), and launched with
// programmatic stream serialization so it may start while its predecessor
// drains (each kernel begins with pdl_wait(); PINT_PDL=0 turns it off).
template <typename... KArgs, typename... Args>
static inline void pint_launch(pint_ctx* ctx, cudaStream_t st, void (*kern)(KArgs...), dim3 grid, dim3 block,
                               size_t smem, Args&&... args) {
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid;
  cfg.blockDim = block;
  cfg.dynamicSmemBytes = smem;
  cfg.stream = counted(ctx, st);
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  // no programmatic edge out of a conditional / memset node or into the first node of a body
  const bool pdl = ctx->pdl && !(ctx->capturing && ctx->nopdl.erase(st));
  attr[0].val.programmaticStreamSerializationAllowed = pdl ? 1 : 0;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  cudaLaunchKernelEx(&cfg, kern, std::forward<Args>(args)...);
}

cudaEvent_t next_event(pint_ctx* ctx) {
  if (ctx->ev_used == ctx->ev_pool.size()) {
    cudaEvent_t e;
    cudaEventCreate(&e);
    ctx->ev_pool.push_back(e);
  }
  return ctx->ev_pool[ctx->ev_used++];
}

#define PINT_CHECK(call)                                                       \
  do {                                                                         \
    cudaError_t e_ = (call);                                                   \
    if (e_ != cudaSuccess) {                                                   \
      ctx->err = std::string(#call) + ": " + cudaGetErrorString(e_);           \
      return PINT_CUDA_ERROR;                                                  \
    }                                                                          \
  } while (0)

#define PINT_LAUNCHED()                                                        \
  do {                                                                         \
    cudaError_t e_ = cudaGetLastError();                                       \
    if (e_ != cudaSuccess) {                                                   \
      ctx->err = std::string("kernel launch: ") + cudaGetErrorString(e_);      \
      return PINT_CUDA_ERROR;                                                  \
    }                                                                          \
  } while (0)

template <typename T>
int dalloc(pint_ctx* ctx, T** p, size_t count) {
  void* q = nullptr;
  cudaError_t e = cudaMalloc(&q, std::max<size_t>(count, 1) * sizeof(T));
  if (e != cudaSuccess) {
    ctx->err = std::string("cudaMalloc(") + std::to_string(count * sizeof(T)) + " B): " + cudaGetErrorString(e);
    return PINT_CUDA_ERROR;
  }
  cudaMemset(q, 0, std::max<size_t>(count, 1) * sizeof(T));
  ctx->allocs.push_back(q);
  ctx->bytes += count * sizeof(T);
  *p = static_cast<T*>(q);
  return PINT_OK;
}

#define PINT_TRY(x)          \
  do {                       \
    int rc_ = (x);           \
    if (rc_ != PINT_OK) return rc_; \
  } while (0)

// ---------------------------------------------------------------- conditional graph capture
// A conditional node is appended to the capture frontier of `st`; its body is
// captured on the next stream of the context's capture-stream stack.  The
// handle lives in the root graph of the capture; `idx` names the body's slot
// in body_nodes (its kernel-node count, for the device launch counter).
int new_cond(pint_ctx* ctx, cudaGraphConditionalHandle* h) {
  PINT_CHECK(cudaGraphConditionalHandleCreate(h, ctx->cap_root, 0, 0));
  if ((int)ctx->body_nodes.size() >= kMaxBodies) {
    ctx->err = "too many conditional bodies (loop-graph cache exhausted)";
    return PINT_CUDA_ERROR;
  }
  ctx->body_nodes.push_back(0);
  return PINT_OK;
}

int capture_cond(pint_ctx* ctx, cudaStream_t st, int depth, cudaGraphConditionalHandle h, bool loop, int idx,
                 const std::function<int(cudaStream_t, int)>& body) {
  if (depth + 1 >= kCapDepth) {
    ctx->err = "conditional nesting too deep";
    return PINT_CUDA_ERROR;
  }
  cudaStreamCaptureStatus cs;
  cudaGraph_t g = nullptr;
  const cudaGraphNode_t* deps = nullptr;
  size_t nd = 0;
  PINT_CHECK(cudaStreamGetCaptureInfo(st, &cs, nullptr, &g, &deps, &nd));
  cudaGraphNodeParams p = {};
  p.type = cudaGraphNodeTypeConditional;
  p.conditional.handle = h;
  p.conditional.type = loop ? cudaGraphCondTypeWhile : cudaGraphCondTypeIf;
  p.conditional.size = 1;
  cudaGraphNode_t node;
  PINT_CHECK(cudaGraphAddNode(&node, g, deps, nd, &p));
  cudaGraph_t bg = p.conditional.phGraph_out[0];
  PINT_CHECK(cudaStreamUpdateCaptureDependencies(st, &node, 1, cudaStreamSetCaptureDependencies));
  ctx->nopdl.insert(st);
  cudaStream_t cst = ctx->cap_st[depth + 1];
  PINT_CHECK(cudaStreamBeginCaptureToGraph(cst, bg, nullptr, nullptr, 0, cudaStreamCaptureModeRelaxed));
  ctx->nopdl.insert(cst);
  const long long before = ctx->launches;
  const int rc = body(cst, depth + 1);
  const long long n = ctx->launches - before;
  ctx->launches = before;
  cudaGraph_t out = nullptr;
  const cudaError_t e = cudaStreamEndCapture(cst, &out);
  if (rc != PINT_OK) return rc;
  PINT_CHECK(e);
  ctx->body_nodes[idx] = (int)n;
  return PINT_OK;
}

Grid make_grid(int dim, const int* cells) {
  Grid g{};
  g.dim = dim;
  g.n[0] = cells[0] + 1;
  g.n[1] = cells[1] + 1;
  g.n[2] = dim == 3 ? cells[2] + 1 : 1;
  g.nn = g.n[0] * g.n[1] * g.n[2];
  g.np = (int)round_up((size_t)g.nn, 32);
  g.C = 2 * dim + 1;
  g.noff = ipow3(dim);
  return g;
}

double ramp_value(double t, double T) {
  const double tt = std::min(t, T);
  return 0.5 * (1.0 - std::cos(M_PI * tt / T));
}

// pressure stabilization delta_K(k); same expression order as FSIProblem.delta_p
double delta_value(const pint_problem_desc& d, double k) {
  double h2 = 0.0;
  for (int m = 0; m < d.dim; ++m) {
    const double h = d.extent[m] / d.cells[m];
    h2 += h * h;
  }
  const double hk = std::sqrt(h2 / d.dim);
  const double tau = d.stab_k > 0.0 ? d.stab_k : hk / d.u_peak;  // k-independent (see FSIProblem.delta_p)
  (void)k;
  return d.alpha_p / (d.rho_f * (1.0 / tau + d.u_peak / hk + d.nu_f / (hk * hk)));
}

StepScalars make_step(const pint_problem_desc& d, double k, double theta, double t1) {
  StepScalars s;
  s.k = k;
  s.kt = k * theta;
  s.ko = k * (1.0 - theta);
  s.ramp = ramp_value(t1, d.ramp_time);
  s.delta = delta_value(d, k);
  return s;
}

inline dim3 node_grid(int nn, int S, int bs = 128) { return dim3((nn + bs - 1) / bs, S); }
inline dim3 row_grid(int nn, int S) { return dim3((nn + 31) / 32, S); }
// enough CTAs to fill the GPU several times: use the lower-register variant
// (3 offsets of loads in flight) for occupancy; small grids put all 9 in flight
inline bool wide(int nn, int S) { return (size_t)((nn + 31) / 32) * S >= 4 * 148; }
template <int D>
inline dim3 row_block() { return dim3(32, 2 * D + 1); }
inline dim3 vec_grid(size_t n, int S) {
  size_t blocks = (n + 255) / 256;
  if (blocks > 1024) blocks = 1024;
  return dim3((unsigned)blocks, S);
}

// ---------------------------------------------------------------- mesh tables (host)
void build_tables(pint_ctx* ctx) {
  const auto& d = ctx->desc;
  const int D = ctx->D;
  const Grid& g = ctx->g;
  const int ncell = ctx->cells[0] * ctx->cells[1] * ctx->cells[2];
  ctx->h_cell_flags.assign(ncell, 0);
  ctx->h_node_flags.assign(g.nn, 0);
  ctx->h_profile.assign(g.nn, 0.0);
  double h[3];
  for (int m = 0; m < 3; ++m) h[m] = m < D ? d.extent[m] / d.cells[m] : 1.0;
  for (int ck = 0; ck < ctx->cells[2]; ++ck)
    for (int cj = 0; cj < ctx->cells[1]; ++cj)
      for (int ci = 0; ci < ctx->cells[0]; ++ci) {
        const int idx[3] = {ci, cj, ck};
        bool solid = true;
        for (int m = 0; m < D; ++m) {
          const double c = (idx[m] + 0.5) * h[m];
          solid = solid && (c >= d.bar_lo[m]) && (c <= d.bar_hi[m]);
        }
        uint8_t f = solid ? kCellSolid : 0;
        if (!solid && ci == ctx->cells[0] - 1) f |= kCellOutflow;
        const int cell = (ck * ctx->cells[1] + cj) * ctx->cells[0] + ci;
        ctx->h_cell_flags[cell] = f;
        for (int a = 0; a < (1 << D); ++a) {
          const int n = node_index(g, ci + (a & 1), cj + ((a >> 1) & 1), D == 3 ? ck + ((a >> 2) & 1) : 0);
          ctx->h_node_flags[n] |= solid ? kSolidTouch : kFluidTouch;
        }
      }
  for (int n = 0; n < g.nn; ++n) {
    int i, j, k;
    node_coords(g, n, i, j, k);
    const int idx[3] = {i, j, k};
    bool wall = false;
    for (int m = 1; m < D; ++m) wall = wall || idx[m] == 0 || idx[m] == d.cells[m];
    const bool in_lo = i == 0, out_hi = i == d.cells[0];
    uint8_t f = ctx->h_node_flags[n];
    if (in_lo || wall) f |= kDirV;
    if (in_lo || out_hi || wall) f |= kDirU;
    ctx->h_node_flags[n] = f;
    double prof = d.u_peak;
    for (int m = 1; m < D; ++m) {
      const double y = idx[m] * h[m];
      const double H = d.extent[m];
      prof = prof * 4.0 * y * (H - y) / (H * H);
    }
    ctx->h_profile[n] = (in_lo && !wall) ? prof : 0.0;
  }
}

// ---------------------------------------------------------------- dimension-specific implementation
template <int D>
struct Impl {
  static constexpr int C = 2 * D + 1;

  static MeshDev mesh(pint_ctx* ctx) {
    MeshDev m;
    m.g = ctx->g;
    m.cells[0] = ctx->cells[0];
    m.cells[1] = ctx->cells[1];
    m.cells[2] = ctx->cells[2];
    m.cell_flags = ctx->d_cell_flags;
    m.node_flags = ctx->d_node_flags;
    m.profile = ctx->d_profile;
    return m;
  }

  static int colour_count(pint_ctx* ctx, int colour) {
    int n = 1;
    for (int m = 0; m < D; ++m) n *= (ctx->cells[m] - ((colour >> m) & 1) + 1) >> 1;
    return n;
  }

  static size_t vs(pint_ctx* ctx) { return (size_t)C * ctx->g.np; }

  // ---- residual r = R(y; yo); norms into ctx->d_norms (and host if h != nullptr)
  static int residual(pint_ctx* ctx, int S, const double* y, const double* yo, double* r, const int* mask,
                      double* h_norms, cudaStream_t st) {
    MeshDev m = mesh(ctx);
    if constexpr (D == 2) {
      if (ctx->res_strip) {
        // node-owner strips: every residual row written once (fixed rows included), one launch
        static bool attr = false;
        if (!attr) {
          cudaFuncSetAttribute(k_residual_strip, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ResStrip::smem);
          attr = true;
        }
        cudaMemsetAsync(ctx->d_degen, 0, sizeof(int) * S, st);
        if (ctx->capturing) ctx->nopdl.insert(st);  // memset node: no programmatic edge out of it
        const int nxn = ctx->cells[0] + 1, nyn = ctx->cells[1] + 1;
        const int wmax = std::max(1, std::min(ctx->strip_w, (int)ResStrip::WMAX));
        const int nstrips = (nxn + wmax - 1) / wmax;
        const int W = (nxn + nstrips - 1) / nstrips;
        const int base = nstrips * S;
        int nch = std::max(1, std::min((ctx->res_waves * 3 * 148 + base - 1) / base, std::max(1, nyn / 2)));
        const int H = (nyn + nch - 1) / nch;
        nch = (nyn + H - 1) / H;
        pint_launch(ctx, st, k_residual_strip, dim3(nstrips * nch, S), ResStrip::T, ResStrip::smem, m, ctx->ph,
                    (const StepScalars*)ctx->d_st, y, yo, r, ctx->d_degen, mask, W, nstrips, H);
        PINT_LAUNCHED();
        return norms(ctx, S, r, r, mask, true, ctx->d_degen, h_norms, st);
      }
    }
    pint_launch(ctx, st, k_zero_active, vec_grid(vs(ctx), S), 256, 0, r, vs(ctx), mask);
    cudaMemsetAsync(ctx->d_degen, 0, sizeof(int) * S, st);
    if (ctx->capturing) ctx->nopdl.insert(st);  // memset node: no programmatic edge out of it
    for (int c = 0; c < (1 << D); ++c) {
      const int ne = colour_count(ctx, c);
      if (ne == 0) continue;
      if (ctx->elem_old)
        pint_launch(ctx, st, k_residual_colour<D>, dim3((ne * (1 << D) + 127) / 128, S), 128, 0, m, ctx->ph,
                    ctx->d_st, y, yo, r, ctx->d_degen, mask, c);
      else
        pint_launch(ctx, st, k_elem_tile<D, 0>, dim3((ne + ElemTile<D>::EPB - 1) / ElemTile<D>::EPB, S),
                    ElemTile<D>::T, ElemTile<D>::smem(2), m, ctx->ph, (const StepScalars*)ctx->d_st, y, yo,
                    (const double*)nullptr, r, ctx->d_degen, mask, c);
    }
    pint_launch(ctx, st, k_fix_residual<D>, node_grid(ctx->g.nn, S), 128, 0, m, ctx->d_st, y, r, mask);
    PINT_LAUNCHED();
    return norms(ctx, S, r, r, mask, true, ctx->d_degen, h_norms, st);
  }

  static int norms(pint_ctx* ctx, int S, const double* x, const double* y, const int* mask, bool take_sqrt,
                   const int* degen, double* h_out, cudaStream_t st) {
    const int nblk = ctx->nblk;
    pint_launch(ctx, st, k_dot_partial, dim3(nblk, S), kRedThreads, 0, x, y, vs(ctx), ctx->partial, nblk, mask);
    pint_launch(ctx, st, k_dot_final, (S + 127) / 128, 128, 0, ctx->partial, nblk, ctx->d_norms, S, take_sqrt ? 1 : 0, degen,
                                                mask);
    PINT_LAUNCHED();
    if (h_out) {
      PINT_CHECK(cudaMemcpyAsync(ctx->h_dbl, ctx->d_norms, sizeof(double) * S, cudaMemcpyDeviceToHost, st));
      PINT_CHECK(cudaStreamSynchronize(st));
      std::memcpy(h_out, ctx->h_dbl, sizeof(double) * S);
    }
    return PINT_OK;
  }

  // ---- Jacobian assembly into level 0
  static int assemble(pint_ctx* ctx, int S, const double* y, const double* yo, const int* mask, cudaStream_t st) {
    MeshDev m = mesh(ctx);
    Level& L0 = ctx->lv[0];
    const size_t ms = (size_t)ctx->g.noff * C * C * ctx->g.np;
    if constexpr (D == 2) {
      if (ctx->jac_strip && !ctx->jac_columns) {
        // node-owner strips: every stencil row written once (fp64 + fp32 copy, fixed rows included)
        static bool attr = false;
        if (!attr) {
          cudaFuncSetAttribute(k_jacobian_strip<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)JacStrip::smem);
          cudaFuncSetAttribute(k_jacobian_strip<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)JacStrip::smem);
          attr = true;
        }
        const int nxn = ctx->cells[0] + 1, nyn = ctx->cells[1] + 1;
        // owned node columns per strip: <= 25 keeps the W * C phase-2 items of a row within one round of the
        // 128 threads (31 needs two, the second nearly empty); PINT_STRIP_W overrides
        const int wmax = std::max(1, std::min(ctx->strip_w, (int)JacStrip::WMAX));
        const int nstrips = (nxn + wmax - 1) / wmax;
        const int W = (nxn + nstrips - 1) / nstrips;
        // enough blocks for ~8 waves at 3 CTAs/SM; each chunk recomputes one halo cell row
        const int base = nstrips * C * S;
        int nch = std::max(1, std::min((8 * 3 * 148 + base - 1) / base, std::max(1, nyn / 4)));
        const int H = (nyn + nch - 1) / nch;
        nch = (nyn + H - 1) / H;
        if (ctx->jac_mt)  // all 1 + d directions of a column component in one multi-tangent flux pass (PINT_JAC_MT=0: one pass each)
          pint_launch(ctx, st, k_jacobian_strip<true>, dim3(nstrips * nch, C, S), JacStrip::T, JacStrip::smem, m, ctx->ph,
                      (const StepScalars*)ctx->d_st, y, yo, L0.A, L0.A32, mask, W, nstrips, H);
        else
          pint_launch(ctx, st, k_jacobian_strip<false>, dim3(nstrips * nch, C, S), JacStrip::T, JacStrip::smem, m, ctx->ph,
                      (const StepScalars*)ctx->d_st, y, yo, L0.A, L0.A32, mask, W, nstrips, H);
        PINT_LAUNCHED();
        return PINT_OK;
      }
    }
    pint_launch(ctx, st, k_zero_active, vec_grid(ms, S), 256, 0, L0.A, ms, mask);
    constexpr int A = 1 << D;
    if (!ctx->jac_columns) {
      using JL = JacLin<D>;
      static bool attr = false;
      if (!attr) {
        cudaFuncSetAttribute(k_jacobian_lin<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)JL::smem);
        attr = true;
      }
      for (int c = 0; c < A; ++c) {
        const int ne = colour_count(ctx, c);
        if (ne == 0) continue;
        pint_launch(ctx, st, k_jacobian_lin<D>, dim3((ne + JL::EPB - 1) / JL::EPB, C, S), JL::T, JL::smem, 
            m, ctx->ph, ctx->d_st, y, yo, L0.A, mask, c);
      }
    } else {
      for (int c = 0; c < A; ++c) {
        const int ne = colour_count(ctx, c);
        if (ne == 0) continue;
        pint_launch(ctx, st, k_jacobian_colour<D>, dim3((ne * A + 127) / 128, A * C, S), 128, 0, m, ctx->ph, ctx->d_st, y, yo, L0.A, mask,
                                                                           c);
      }
    }
    pint_launch(ctx, st, k_fix_jacobian<D>, node_grid(ctx->g.nn, S), 128, 0, m, L0.A, mask);
    if (L0.A32) pint_launch(ctx, st, k_to_f32, vec_grid(ms / 2, S), 256, 0, L0.A, L0.A32, ms, mask);
    PINT_LAUNCHED();
    return PINT_OK;
  }

  // the shared-memory staged fp32 residual kernel runs on this level
  static bool resid_staged(const pint_ctx* ctx, const Level& L, int S) {
    return L.A32 && ctx->spmv32_staged && (size_t)L.g.nn * S >= ctx->spmv32_min;
  }

  // V-cycle residual r = b - A x on level L (fp32 operator copy on level 0 when present)
  static void vc_resid(pint_ctx* ctx, const Level& L, int S, const double* x, const double* b, double* r,
                       const int* mask, cudaStream_t st) {
    const bool w = wide(L.g.nn, S);
    // node-per-thread kernel once the level fills >= 2 waves of 128-thread
    // CTAs (c3 levels 0-1: +4.6 %); below that the (node, row) threads hide
    // latency better (c2, L2-resident: -3 % with the node kernel)
    if (resid_staged(ctx, L, S)) {
      if (ctx->resid_acc32)
        pint_launch(ctx, st, k_resid32_staged<D, false, true>, row_grid(L.g.nn, S), dim3(32, D + 2), 0, L.g,
                    (const float*)L.A32, x, b, r, mask, L.g, (const double*)nullptr, (double*)nullptr);
      else
        pint_launch(ctx, st, k_resid32_staged<D, false>, row_grid(L.g.nn, S), dim3(32, D + 2), 0, L.g,
                    (const float*)L.A32, x, b, r, mask, L.g, (const double*)nullptr, (double*)nullptr);
    } else if (L.A32 && ctx->spmv32_node && (size_t)L.g.nn * S >= ctx->spmv32_min) {
      pint_launch(ctx, st, k_spmv_node<D, true, float>, node_grid(L.g.nn, S), 128, 0, L.g, (const float*)L.A32, x, b, r,
                  mask);
    } else if (L.A32) {
      if (w) pint_launch(ctx, st, k_spmv<D, true, 3, float>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.A32, x, b, r, mask);
      else pint_launch(ctx, st, k_spmv<D, true, 9, float>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.A32, x, b, r, mask);
    } else {
      if (w) pint_launch(ctx, st, k_spmv<D, true, 3>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.A, x, b, r, mask);
      else pint_launch(ctx, st, k_spmv<D, true, 9>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.A, x, b, r, mask);
    }
  }

  static int jvp(pint_ctx* ctx, int S, const double* y, const double* yo, const double* w, double* out,
                 cudaStream_t st) {
    MeshDev m = mesh(ctx);
    pint_launch(ctx, st, k_zero_active, vec_grid(vs(ctx), S), 256, 0, out, vs(ctx), nullptr);
    for (int c = 0; c < (1 << D); ++c) {
      const int ne = colour_count(ctx, c);
      if (ne == 0) continue;
      if (ctx->elem_old)
        pint_launch(ctx, st, k_jvp_colour<D>, dim3((ne * (1 << D) + 127) / 128, S), 128, 0, m, ctx->ph,
                    ctx->d_st, y, yo, w, out, nullptr, c);
      else
        pint_launch(ctx, st, k_elem_tile<D, 1>, dim3((ne + ElemTile<D>::EPB - 1) / ElemTile<D>::EPB, S),
                    ElemTile<D>::T, ElemTile<D>::smem(3), m, ctx->ph, (const StepScalars*)ctx->d_st, y, yo, w,
                    out, (int*)nullptr, (const int*)nullptr, c);
    }
    pint_launch(ctx, st, k_fix_jvp<D>, node_grid(ctx->g.nn, S), 128, 0, m, w, out, nullptr);
    PINT_LAUNCHED();
    return PINT_OK;
  }

  static void spmv(pint_ctx* ctx, int lvl, int S, const double* x, double* y, const int* mask, cudaStream_t st) {
    Level& L = ctx->lv[lvl];
    if (wide(L.g.nn, S))
      pint_launch(ctx, st, k_spmv<D, false, 3>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.A, x, nullptr, y, mask);
    else
      pint_launch(ctx, st, k_spmv<D, false, 9>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.A, x, nullptr, y, mask);
  }

  // ---- multigrid setup: RAP on all levels, block inverses, dense coarsest
  static int precond_setup(pint_ctx* ctx, int S, const pint_krylov_opts* ko, const int* mask, cudaStream_t st) {
    int nl = (int)ctx->lv.size();
    if (ko->max_levels > 0) {
      nl = std::min(nl, (int)ko->max_levels);
    } else {
      // default: stop at the first level the cluster Gauss-Jordan inverts; a
      // dense solve there replaces the latency-bound sweeps of the levels below
      for (int l = 0; l < nl; ++l)
        if (C * ctx->lv[l].g.nn <= ctx->dense_cap && gj_fits(C * ctx->lv[l].g.nn)) {
          nl = l + 1;
          break;
        }
    }
    ctx->prec_levels = nl;
    ctx->kopt = *ko;
    // coarsest used level solved with a dense inverse when it fits the buffer
    ctx->dense_n = C * ctx->lv[nl - 1].g.nn;
    ctx->coarse_dense = ctx->d_dense != nullptr && ctx->dense_n <= ctx->dense_cap;
    for (int l = 0; l < nl; ++l) {
      Level& L = ctx->lv[l];
      if (l > 0) {
        Level& F = ctx->lv[l - 1];
        pint_launch(ctx, st, k_rap<D>, dim3((L.g.nn + 63) / 64, L.g.noff * C, S), 64, 0, F.g, L.g, F.A, L.A, mask);
        if (L.A32) {
          const size_t ms = (size_t)L.g.noff * C * C * L.g.np;
          pint_launch(ctx, st, k_to_f32, vec_grid(ms / 2, S), 256, 0, (const double*)L.A, L.A32, ms, mask);
        }
      }
      const bool last_dense = ctx->coarse_dense && l == nl - 1;
      if (ko->smoother == 1 && !last_dense && !ctx->vanka_smem) {
        using VR = VankaRows<D>;
        pint_launch(ctx, st, k_vanka_setup_rows<D>, dim3((L.ncell + VR::CPB - 1) / VR::CPB, S), VR::T, 0, 
            L.g, L.A, L.vinv, mask);
      } else if (ko->smoother == 1 && !last_dense) {
        constexpr int W = D == 2 ? 4 : 2;
        constexpr int Lc = Cells<D>::L;
        const size_t smem = (size_t)W * (Lc * 2 * Lc + Lc) * sizeof(double);
        cudaFuncSetAttribute(k_vanka_setup<D, W>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        pint_launch(ctx, st, k_vanka_setup<D, W>, dim3((L.ncell + W - 1) / W, S), 32 * W, smem, L.g, L.A, L.vinv,
                                                                                                mask);
      } else {
        pint_launch(ctx, st, k_block_inverse<D>, node_grid(L.g.nn, S), 128, 0, L.g, L.A, L.Dinv, mask);
      }
      // block-stencil form of the sweep on the levels that run standalone kernels
      if (ko->smoother == 1 && !last_dense && ctx->vanka_stencil && L.vst)
        pint_launch(ctx, st, k_vanka_stencil_build<D>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g,
                    (const float*)L.vinv, L.vst, (double)ko->omega, mask);
    }
    if (ctx->coarse_dense) {
      Level& L = ctx->lv[nl - 1];
      const int n = ctx->dense_n;
      ctx->dense_ld = (n + 3) / 4 * 4;
      const size_t smem = gj_smem_bytes(n);
      if (gj_fits(n)) {
        cudaFuncSetAttribute(k_dense_invert_cl<D>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
        pint_launch(ctx, st, k_dense_invert_cl<D>, S * kGJCluster, kGJThreads, smem, L.g, L.A, ctx->d_dense32, n,
                                                                                      ctx->dense_ld, mask);
      } else {
        pint_launch(ctx, st, k_dense_build<D>, dim3(1, S), 512, 0, L.g, L.A, ctx->d_dense, mask);
        pint_launch(ctx, st, k_gauss_jordan, S, 512, 0, ctx->d_dense, n, mask);
        pint_launch(ctx, st, k_dense_to_f32, dim3((n * n + 255) / 256, S), 256, 0, ctx->d_dense, ctx->d_dense32, n,
                                                                                 ctx->dense_ld, mask);
      }
    }
    // fused V-cycle tail: from the first level with <= 2048 rows per slice down
    ctx->tail_first = -1;
    if (ctx->use_tail && ko->smoother == 1 && nl <= kMaxLevels) {
      for (int l = 0; l < nl; ++l)
        if ((size_t)ctx->lv[l].g.nn * C <= (size_t)ctx->tail_rows) { ctx->tail_first = l; break; }
      if (ctx->tail_first >= 0) {
        TailArgs& t = ctx->tail;
        for (int l = 0; l < nl; ++l) {
          Level& L = ctx->lv[l];
          t.lv[l] = LevelDev{L.g, L.A, L.vinv, ctx->vanka_stencil ? L.vst : nullptr, L.rhs, L.xa, L.xb, L.res, L.sol, L.ycell, L.ncell};
        }
        t.first = ctx->tail_first;
        t.last = nl - 1;
        t.dense = ctx->coarse_dense ? ctx->d_dense32 : nullptr;
        t.dense_ld = ctx->dense_ld;
        // cluster tails: each CTA stages its rows of the inverse when they fit shared memory
        t.dense_stage = 0;
        if (ctx->coarse_dense) {
          const int n = ctx->dense_n, ld = ctx->dense_ld;
          const size_t t8 = tail_dense_smem(n, ld, 8), t4 = tail_dense_smem(n, ld, 4), t2 = tail_dense_smem(n, ld, 2);
          if (t8 <= kTailSmemMax)
            cudaFuncSetAttribute(k_vcycle_tail_cl<D, 8>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t8);
          if (t4 <= kTailSmemMax)
            cudaFuncSetAttribute(k_vcycle_tail_cl<D, 4>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t4);
          if (t2 <= kTailSmemMax)
            cudaFuncSetAttribute(k_vcycle_tail_cl<D, 2>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)t2);
        }
        t.coarse_sweeps = ko->coarse_sweeps;
        t.pre = ko->pre_smooth;
        t.post = ko->post_smooth;
        t.omega = ko->omega;
        ctx->tail_cl = t;
        ctx->tail_cl.dense_stage = ctx->coarse_dense ? 1 : 0;
      }
    }
    // fused Arnoldi step: the whole step in one cluster launch per slice when
    // the level-0 grid is small (a property of the mesh, never of the batch)
    ctx->fused = ctx->use_fused && ctx->tail_first >= 0 && (size_t)ctx->lv[0].g.nn * C <= kFusedRows &&
                 ctx->restart + 1 <= kMaxBasis;
    if (ctx->fused) {
      ctx->tail0 = ctx->tail;
      ctx->tail0.first = 0;
    }
    PINT_LAUNCHED();
    return PINT_OK;
  }

  // resid_done: L.res already holds b - A xin (the fused prolongation + residual kernel)
  static void smooth(pint_ctx* ctx, const Level& L, int S, const double* b, const double* xin, double* xout,
                     const int* mask, cudaStream_t st, bool first, bool resid_done = false) {
    const double om = ctx->kopt.omega;
    if (ctx->kopt.smoother == 1) {
      constexpr int CELLS = D == 2 ? 16 : 8;
      const double* r = b;
      if (!first) {
        if (!resid_done) vc_resid(ctx, L, S, xin, b, L.res, mask, st);
        r = L.res;
      }
      const bool prof = ctx->prof && &L == &ctx->lv[0];
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (prof) {
        e0 = next_event(ctx);
        e1 = next_event(ctx);
        cudaEventRecord(e0, st);
      }
      if (ctx->vanka_stencil && L.vst) {
        // the sweep as one fp32 block-stencil product (k_vanka_stencil_build at the hierarchy build)
        if (first && ctx->defer_w && &L == &ctx->lv[0]) {
          pint_launch(ctx, st, k_vanka_stencil_apply<D, true>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g,
                      (const float*)L.vst, (const double*)ctx->defer_w, nullptr, xout, mask,
                      prof ? ctx->d_work : nullptr, (const double*)ctx->defer_w, (const double*)ctx->gm_hnorm,
                      const_cast<double*>(b));
          ctx->defer_w = nullptr;
        } else if (first)
          pint_launch(ctx, st, k_vanka_stencil_apply<D, true>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g,
                      (const float*)L.vst, r, nullptr, xout, mask, prof ? ctx->d_work : nullptr, nullptr, nullptr,
                      nullptr);
        else
          pint_launch(ctx, st, k_vanka_stencil_apply<D, false>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g,
                      (const float*)L.vst, r, xin, xout, mask, prof ? ctx->d_work : nullptr, nullptr, nullptr,
                      nullptr);
        if (prof) {
          cudaEventRecord(e1, st);
          ctx->ev_pairs.emplace_back(e0, e1);
        }
        return;
      }
      if (!ctx->vanka_split) {
        // fused cell solves + gather (bitwise the same as the split pair below)
        if (first && ctx->defer_w && &L == &ctx->lv[0]) {
          // b = v_j is formed from the previous step's unscaled w inside the sweep
          pint_launch(ctx, st, k_vanka_apply<D, true>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.vinv,
                      (const double*)ctx->defer_w, nullptr, xout, om, mask, prof ? ctx->d_work : nullptr,
                      (const double*)ctx->defer_w, (const double*)ctx->gm_hnorm, const_cast<double*>(b));
          ctx->defer_w = nullptr;
        } else if (first)
          pint_launch(ctx, st, k_vanka_apply<D, true>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.vinv, r,
                      nullptr, xout, om, mask, prof ? ctx->d_work : nullptr, nullptr, nullptr, nullptr);
        else
          pint_launch(ctx, st, k_vanka_apply<D, false>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.vinv, r,
                      xin, xout, om, mask, prof ? ctx->d_work : nullptr, nullptr, nullptr, nullptr);
        if (prof) {
          cudaEventRecord(e1, st);
          ctx->ev_pairs.emplace_back(e0, e1);
        }
        return;
      }
      pint_launch(ctx, st, k_vanka_cell<D, CELLS>, dim3((L.ncell + CELLS - 1) / CELLS, S), dim3(CELLS, Cells<D>::L), 0, 
          L.g, L.vinv, r, L.ycell, mask, prof ? ctx->d_work : nullptr);
      if (prof) {
        cudaEventRecord(e1, st);
        ctx->ev_pairs.emplace_back(e0, e1);
      }
      if (first)
        pint_launch(ctx, st, k_vanka_gather<D, true>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.ycell, nullptr,
                                                                                              xout, om, mask);
      else
        pint_launch(ctx, st, k_vanka_gather<D, false>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.ycell, xin,
                                                                                               xout, om, mask);
      return;
    }
    if (first) {
      pint_launch(ctx, st, k_smooth<D, true, 3>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, L.A, L.Dinv, b, nullptr,
                                                                                    xout, om, mask, nullptr);
      return;
    }
    const bool prof = ctx->prof && &L == &ctx->lv[0];
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (prof) {
      e0 = next_event(ctx);
      e1 = next_event(ctx);
      cudaEventRecord(e0, st);
    }
    if (wide(L.g.nn, S))
      pint_launch(ctx, st, k_smooth<D, false, 3>, row_grid(L.g.nn, S), row_block<D>(), 0, 
          L.g, L.A, L.Dinv, b, xin, xout, om, mask, prof ? ctx->d_work : nullptr);
    else
      pint_launch(ctx, st, k_smooth<D, false, 9>, row_grid(L.g.nn, S), row_block<D>(), 0, 
          L.g, L.A, L.Dinv, b, xin, xout, om, mask, prof ? ctx->d_work : nullptr);
    if (prof) {
      cudaEventRecord(e1, st);
      ctx->ev_pairs.emplace_back(e0, e1);
    }
  }

  // x = V-cycle(b) on level l; b and x must not alias level scratch of l
  static void vcycle(pint_ctx* ctx, int l, int S, const double* b, double* x, const int* mask, cudaStream_t st) {
    Level& L = ctx->lv[l];
    const int nl = ctx->prec_levels;
    const pint_krylov_opts& ko = ctx->kopt;
    if (l == ctx->tail_first) {
      // whole V-cycle inside the tail kernel (small meshes): it is the profiled kernel
      const bool prof = ctx->prof && l == 0;
      cudaEvent_t e0 = nullptr, e1 = nullptr;
      if (prof) {
        e0 = next_event(ctx);
        e1 = next_event(ctx);
        cudaEventRecord(e0, st);
        ctx->tail_slice_launches += S;
      }
      const int cl = tail_cluster_size(ctx, S);
      const size_t tsm = ctx->coarse_dense ? tail_dense_smem(ctx->dense_n, ctx->dense_ld, cl) : 0;
      // the coarsest inverse is staged in shared memory whenever a CTA's rows fit, even when that runs the
      // S * cl CTAs in two waves (c3, S = 64, cl = 4: 929 staged vs 887 from L2; c2 8438 vs 6341);
      // PINT_TAIL_STAGE=0 reads it from L2
      const bool stage = ctx->coarse_dense && tsm <= kTailSmemMax && ctx->tail_stage != 0;
      const TailArgs& ta = stage ? ctx->tail_cl : ctx->tail;
      const size_t sm = stage ? tsm : 0;
      if (cl == 8)
        pint_launch(ctx, st, k_vcycle_tail_cl<D, 8>, S * 8, kTailThreads, sm, ta, b, x, mask);
      else if (cl == 4)
        pint_launch(ctx, st, k_vcycle_tail_cl<D, 4>, S * 4, kTailThreads, sm, ta, b, x, mask);
      else if (cl == 2)
        pint_launch(ctx, st, k_vcycle_tail_cl<D, 2>, S * 2, kTailThreads, sm, ta, b, x, mask);
      else
        pint_launch(ctx, st, k_vcycle_tail<D>, S, 1024, 0, ctx->tail, b, x, mask);
      if (prof) {
        cudaEventRecord(e1, st);
        ctx->ev_pairs.emplace_back(e0, e1);
      }
      return;
    }
    if (l == nl - 1) {
      if (ctx->coarse_dense) {
        pint_launch(ctx, st, k_dense_apply<D>, S, 256, 0, L.g, ctx->d_dense32, ctx->dense_ld, b, x, mask);
      } else {
        const int sweeps = std::max(1, (int)ko.coarse_sweeps);
        double* cur = L.xa;
        double* nxt = L.xb;
        smooth(ctx, L, S, b, nullptr, sweeps == 1 ? x : cur, mask, st, true);
        for (int i = 1; i < sweeps; ++i) {
          double* out = (i == sweeps - 1) ? x : nxt;
          smooth(ctx, L, S, b, cur, out, mask, st, false);
          std::swap(cur, nxt);
        }
      }
      return;
    }
    Level& Lc = ctx->lv[l + 1];
    const int pre = std::max(1, (int)ko.pre_smooth);
    const int post = std::max(1, (int)ko.post_smooth);
    double* cur = L.xa;
    double* nxt = L.xb;
    smooth(ctx, L, S, b, nullptr, cur, mask, st, true);
    for (int i = 1; i < pre; ++i) {
      smooth(ctx, L, S, b, cur, nxt, mask, st, false);
      std::swap(cur, nxt);
    }
    vc_resid(ctx, L, S, cur, b, L.res, mask, st);
    pint_launch(ctx, st, k_restrict<D>, row_grid(Lc.g.nn, S), row_block<D>(), 0, L.g, Lc.g, L.res, Lc.rhs, mask);
    double* xc = Lc.sol;
    vcycle(ctx, l + 1, S, Lc.rhs, xc, mask, st);
    if (ctx->fuse_prolong && post == 1 && ko.smoother == 1 && resid_staged(ctx, L, S)) {
      // coarse-grid correction inside the post-smoothing residual: x' = cur + P xc goes to nxt (out of
      // place), L.res = b - A x' (bitwise k_prolong_add + the plain residual; PINT_FUSE_PROLONG=1, off by default)
      pint_launch(ctx, st, k_resid32_staged<D, true>, row_grid(L.g.nn, S), dim3(32, D + 2), 0, L.g,
                  (const float*)L.A32, (const double*)cur, b, L.res, mask, Lc.g, (const double*)xc, nxt);
      smooth(ctx, L, S, b, nxt, x, mask, st, false, true);
      return;
    }
    pint_launch(ctx, st, k_prolong_add<D>, row_grid(L.g.nn, S), row_block<D>(), 0, L.g, Lc.g, xc, cur, mask);
    for (int i = 0; i < post; ++i) {
      double* out = (i == post - 1) ? x : nxt;
      smooth(ctx, L, S, b, cur, out, mask, st, false);
      std::swap(cur, nxt);
    }
  }

  // one Arnoldi step j of GMRES for the slices in gm_active (device mask):
  // z = M^{-1} v_j, w = J z, CGS2 against v_0..v_j, h_{j+1,j} = ||w||,
  // v_{j+1} = w / h_{j+1,j}, Givens update.  Every scalar it needs lives in
  // device memory, so the sequence is captured once per (S, j, options) as
  // a CUDA graph and replayed.
  //
  // front: z_j = M^{-1} v_j (flexible GMRES keeps z_j, so the update x += Z y
  // needs no extra V-cycle), w = J z_j; returns whether v_{j+1} = w / h is
  // deferred into the next step's first level-0 Vanka sweep
  static bool arnoldi_front(pint_ctx* ctx, int S, int j, cudaStream_t st) {
    const size_t vstride = (size_t)ctx->maxS * vs(ctx);
    double* vj = ctx->V + j * vstride;
    double* zj = ctx->Z + j * vstride;
    if (ctx->matrix_free) {  // z_j = v_j (Z aliases V), w = J(y) v_j by the K2' kernel
      jvp(ctx, S, ctx->mf_y, ctx->mf_yo, vj, ctx->w, st);
      return false;
    }
    // v_j = w / h_{j,j-1} deferred into the first smoothing sweep of this
    // step's V-cycle (level 0 outside the tail, fused 2-d Vanka sweep)
    const bool defer = ctx->defer_scale && ctx->kopt.smoother == 1 && !ctx->vanka_split && ctx->tail_first != 0 &&
                       !(ctx->prec_levels == 1 && ctx->coarse_dense) && ctx->scale_fuse_max == 0;
    ctx->defer_w = (defer && j >= 1) ? ctx->w : nullptr;
    vcycle(ctx, 0, S, vj, zj, ctx->gm_active, st);
    ctx->defer_w = nullptr;
    spmv(ctx, 0, S, zj, ctx->w, ctx->gm_active, st);
    return defer;
  }

  // Gram-Schmidt dots of pass `pass` (h = <V, w>; pass 1 into ybuf and h += ybuf)
  static void cgs_mdot(pint_ctx* ctx, int S, int j, int pass, const int* act2, cudaStream_t st) {
    const int m = ctx->restart;
    const size_t n = vs(ctx);
    const size_t vstride = (size_t)ctx->maxS * n;
    double* hcol = ctx->H + (size_t)j * (m + 1);
    const int hstride = (m + 1) * m;
    const int nblk = ctx->nblk;
    // wide grids: one block per chunk reading w once; narrow grids (c1/c2): one block per (chunk, vector)
    if ((size_t)nblk * S >= 2 * 148)
      pint_launch(ctx, st, k_mdot_fused, dim3(nblk, S), kRedThreads, 0, ctx->V, vstride, ctx->w, j + 1, n,
                  ctx->partial, nblk, m + 1, hcol, hstride, pass, ctx->ybuf, m + 1, ctx->ctr_mdot, ctx->gm_active,
                  act2);
    else
      pint_launch(ctx, st, k_mdot_fused_v, dim3(nblk, j + 1, S), kRedThreads, 0, ctx->V, vstride, ctx->w, j + 1, n,
                  ctx->partial, nblk, m + 1, hcol, hstride, pass, ctx->ybuf, m + 1, ctx->ctr_mdot, ctx->gm_active,
                  act2);
  }

  // w -= sum_v c_v V_v with the pass's coefficients (h after pass 0, ybuf after pass 1)
  static void cgs_update(pint_ctx* ctx, int S, int j, int pass, const int* mask2, cudaStream_t st) {
    const int m = ctx->restart;
    const size_t n = vs(ctx);
    const size_t vstride = (size_t)ctx->maxS * n;
    double* hcol = ctx->H + (size_t)j * (m + 1);
    const int hstride = (m + 1) * m;
    pint_launch(ctx, st, k_mupdate, vec_grid(n, S), 256, 0, ctx->w, ctx->V, vstride, pass == 0 ? hcol : ctx->ybuf,
                pass == 0 ? hstride : (m + 1), j + 1, n, ctx->gm_active, mask2);
  }

  // h_{j+1,j} = ||w||, Givens update (last block per slice), v_{j+1} = w / h_{j+1,j}
  // (optionally the scaling inside the last block when a slice is small);
  // two: per-slice second-pass flags (nullptr: every slice ran one pass)
  static void arnoldi_tail(pint_ctx* ctx, int S, int j, const int* two, bool defer, cudaStream_t st) {
    const int m = ctx->restart;
    const size_t n = vs(ctx);
    const size_t vstride = (size_t)ctx->maxS * n;
    double* hcol = ctx->H + (size_t)j * (m + 1);
    const int hstride = (m + 1) * m;
    const int nblk = ctx->nblk;
    double* vj1 = ctx->V + (j + 1) * vstride;
    const bool fuse_scale = !ctx->split_norm && n <= (size_t)ctx->scale_fuse_max;
    if (ctx->split_norm)
      pint_launch(ctx, st, k_norm_givens, dim3(nblk, S), kRedThreads, 0, ctx->w, n, ctx->partial, nblk, j, m, ctx->H,
                  ctx->cs, ctx->sn, ctx->gv, ctx->gm_tol, ctx->gm_active, ctx->gm_steps, ctx->gm_its, ctx->gm_res,
                  ctx->gm_hnorm, ctx->ctr_norm, (const int*)ctx->gm_cap);
    else  // last Gram-Schmidt update fused with the norm + Givens (same bits)
      pint_launch(ctx, st, k_mupdate_norm_givens, dim3(nblk, S), kRedThreads, 0, ctx->w, ctx->V, vstride, hcol,
                  hstride, ctx->ybuf, m + 1, two, j + 1, n, ctx->partial, nblk, j, m, ctx->H, ctx->cs, ctx->sn,
                  ctx->gv, ctx->gm_tol, ctx->gm_active, ctx->gm_steps, ctx->gm_its, ctx->gm_res, ctx->gm_hnorm,
                  ctx->ctr_norm, fuse_scale ? vj1 : nullptr, (const int*)ctx->gm_cap);
    if (!fuse_scale && !defer)  // deferred: step j+1 forms v_{j+1} (unused when j+1 == m)
      pint_launch(ctx, st, k_scale_inv, vec_grid(n, S), 256, 0, vj1, ctx->w, ctx->gm_hnorm, n, ctx->gm_active);
  }

  static void arnoldi_step(pint_ctx* ctx, int S, int j, cudaStream_t st) {
    const bool defer = arnoldi_front(ctx, S, j, st);
    // Gram-Schmidt passes: cur_passes = 2 when any slice of the solve wants a
    // second pass; then the pass-1 kernels are masked to those slices
    // (gm_two_pass) and the others subtract their first-pass coefficients in
    // the fused norm kernel -- bitwise the one-pass computation, so a slice's
    // result never depends on the other slices of the batch
    const int npass = ctx->cur_passes;
    const int* two = (npass == 2 && !ctx->split_norm) ? ctx->gm_two_pass : nullptr;
    for (int pass = 0; pass < npass; ++pass) {
      cgs_mdot(ctx, S, j, pass, pass == 1 ? two : nullptr, st);
      if (pass == npass - 1 && !ctx->split_norm) break;
      cgs_update(ctx, S, j, pass, pass == 0 ? two : nullptr, st);
    }
    arnoldi_tail(ctx, S, j, npass == 2 ? ctx->gm_two_pass : nullptr, defer, st);
  }

  // the same step inside the device-driven loop: `two` selects the two-pass
  // form (pass-2 kernels masked to the slices that want it, bitwise the
  // one-pass computation for the others)
  static int arnoldi_step_dev(pint_ctx* ctx, int S, int j, bool two, cudaStream_t st) {
    const bool defer = arnoldi_front(ctx, S, j, st);
    cgs_mdot(ctx, S, j, 0, nullptr, st);
    if (two) {
      cgs_update(ctx, S, j, 0, ctx->gm_two_pass, st);
      cgs_mdot(ctx, S, j, 1, ctx->gm_two_pass, st);
    }
    arnoldi_tail(ctx, S, j, ctx->gm_two_pass, defer, st);
    PINT_LAUNCHED();
    return PINT_OK;
  }

  // algorithmic bytes of one V-cycle from level `from` down, for one slice
  static unsigned long long vcycle_bytes(pint_ctx* ctx, int from) {
    unsigned long long total = 0;
    const int nl = ctx->prec_levels;
    const int Lc = (1 << D) * C;
    for (int l = from; l < nl; ++l) {
      const Level& L = ctx->lv[l];
      const unsigned long long V = (unsigned long long)C * 8 * L.g.nn;
      // the V-cycle residuals read the fp32 copy of level 0 when it exists
      // structurally non-zero coefficient planes only (row_couples: the deformation rows hold 2 of C)
      const unsigned long long Ab = (unsigned long long)L.g.noff * (C * C - D * (C - 2)) * (L.A32 ? 4 : 8) * L.g.nn;
      if (l == nl - 1 && ctx->coarse_dense) {
        total += (unsigned long long)ctx->dense_n * ctx->dense_n * 4 + 2 * V;  // fp32 inverse
        continue;
      }
      const unsigned long long cellb = (ctx->vanka_stencil && L.vst && (ctx->tail_first < 0 || l < ctx->tail_first))
                                           ? (unsigned long long)L.g.noff * C * C * 4 * L.g.nn
                                           : (unsigned long long)L.ncell * ((unsigned long long)Lc * Lc * 4 + 2 * Lc * 8);
      // first sweep + (pre-1 + post) full sweeps + restriction residual + transfers
      const int full = ctx->kopt.pre_smooth - 1 + ctx->kopt.post_smooth;
      total += (cellb + 2 * V) + full * (Ab + 2 * V + cellb + 2 * V) + (Ab + 2 * V) + 3 * V;
    }
    return total;
  }

  // algorithmic bytes of one Arnoldi step j for one slice (fused kernel roofline)
  static unsigned long long arnoldi_bytes(pint_ctx* ctx, int j) {
    unsigned long long total = vcycle_bytes(ctx, 0);
    const unsigned long long V0 = (unsigned long long)C * 8 * ctx->lv[0].g.nn;
    const unsigned long long A0 = (unsigned long long)ctx->lv[0].g.noff * (C * C - D * (C - 2)) * 8 * ctx->lv[0].g.nn;
    total += A0 + 2 * V0;                          // w = J z
    total += 2 * (2ULL * (j + 1) * V0 + 2 * V0);   // CGS2: two dot passes + two updates
    total += 3 * V0;                               // norm + scale
    return total;
  }

  static int launch_fused(pint_ctx* ctx, int S, int j, cudaStream_t st) {
    ArnoldiArgs a{};
    a.vc = ctx->tail0;
    a.V = ctx->V;
    a.Z = ctx->Z;
    a.w = ctx->w;
    a.vstride = (size_t)ctx->maxS * vs(ctx);
    a.per_slice = vs(ctx);
    a.H = ctx->H;
    a.cs = ctx->cs;
    a.sn = ctx->sn;
    a.gv = ctx->gv;
    a.tol = ctx->gm_tol;
    a.gm_active = ctx->gm_active;
    a.gm_steps = ctx->gm_steps;
    a.its = ctx->gm_its;
    a.resid = ctx->gm_res;
    a.hnorm = ctx->gm_hnorm;
    a.cap = ctx->gm_cap;
    a.cpart = ctx->cpart;
    a.ybuf = ctx->ybuf;
    a.work_bytes = ctx->prof ? ctx->d_work_bytes : nullptr;
    a.work_count = ctx->prof ? ctx->d_work : nullptr;
    a.bytes_per_slice = arnoldi_bytes(ctx, j);
    a.j = j;
    a.m = ctx->restart;
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (ctx->prof) {
      e0 = next_event(ctx);
      e1 = next_event(ctx);
      cudaEventRecord(e0, st);
      ctx->fused_used = true;
    }
    pint_launch(ctx, st, k_arnoldi_fused<D>, S * kTailCluster, kTailThreads, 0, a);
    if (ctx->prof) {
      cudaEventRecord(e1, st);
      ctx->ev_pairs.emplace_back(e0, e1);
    }
    PINT_LAUNCHED();
    return PINT_OK;
  }

  static int run_arnoldi(pint_ctx* ctx, int S, int j, cudaStream_t st) {
    if (ctx->fused && (!ctx->use_graphs || ctx->prof)) return launch_fused(ctx, S, j, st);
    if (!ctx->use_graphs || ctx->prof || ctx->matrix_free) {
      arnoldi_step(ctx, S, j, st);
      PINT_LAUNCHED();
      return PINT_OK;
    }
    const GraphKey key{S, j, ctx->prec_levels, ctx->kopt.pre_smooth, ctx->kopt.post_smooth, ctx->kopt.coarse_sweeps,
                       ctx->cur_passes * 100000 + ctx->kopt.smoother * 1000 + ctx->tail_first * 10 + (ctx->fused ? 1 : 0),
                       ctx->kopt.omega};
    auto it = ctx->graphs.find(key);
    if (it == ctx->graphs.end()) {
      cudaGraph_t graph;
      const long long before = ctx->launches;
      PINT_CHECK(cudaStreamBeginCapture(st, cudaStreamCaptureModeThreadLocal));
      if (ctx->fused) launch_fused(ctx, S, j, st);
      else arnoldi_step(ctx, S, j, st);
      PINT_CHECK(cudaStreamEndCapture(st, &graph));
      cudaGraphExec_t exec;
      PINT_CHECK(cudaGraphInstantiate(&exec, graph, 0));
      cudaGraphDestroy(graph);
      const long long nodes = ctx->launches - before;
      ctx->launches = before;
      it = ctx->graphs.emplace(key, std::make_pair(exec, nodes)).first;
    }
    PINT_CHECK(cudaGraphLaunch(it->second.first, st));
    ctx->launches += it->second.second;
    return PINT_OK;
  }

  // ---- GMRES(m), right preconditioned:  J x = b  for slices in mask
  static int gmres(pint_ctx* ctx, int S, const double* b, double* x, const int* mask, const pint_krylov_opts* ko,
                   const double* rtol_s, const double* atol_s,
                   int* h_its, double* h_res, cudaStream_t st,
                   const int* h_mask = nullptr, const double* h_beta = nullptr) {
    const int m = ctx->restart;
    const size_t n = vs(ctx);
    const size_t vstride = (size_t)ctx->maxS * n;
    // h_mask / h_beta: the caller's host copy of the mask and of ||b|| (the
    // Newton loop knows both: b = -r, and ||-r|| is bitwise its ||r||), which
    // saves two host round trips per solve
    std::vector<int> host_mask(S, 1);
    if (mask && h_mask) {
      for (int s = 0; s < S; ++s) host_mask[s] = h_mask[s];
    } else if (mask) {
      PINT_CHECK(cudaMemcpyAsync(ctx->h_int, mask, sizeof(int) * S, cudaMemcpyDeviceToHost, st));
      PINT_CHECK(cudaStreamSynchronize(st));
      for (int s = 0; s < S; ++s) host_mask[s] = ctx->h_int[s];
    }
    // x = 0, r = b, beta = ||b||, tol = max(rtol beta0, atol)
    pint_launch(ctx, st, k_zero_active, vec_grid(n, S), 256, 0, x, n, mask);
    if (!h_beta) {
      PINT_TRY(norms(ctx, S, b, b, mask, true, nullptr, nullptr, st));
      PINT_CHECK(cudaMemcpyAsync(ctx->h_dbl, ctx->d_norms, sizeof(double) * S, cudaMemcpyDeviceToHost, st));
      PINT_CHECK(cudaStreamSynchronize(st));
    }
    std::vector<double> beta(S, 0.0), tol(S, 0.0);
    for (int s = 0; s < S; ++s) {
      beta[s] = h_beta ? (host_mask[s] ? h_beta[s] : 0.0) : ctx->h_dbl[s];
      // per-slice stopping test: ||r|| <= max(rtol_s beta, atol_s) (defaults: the options)
      tol[s] = std::max((rtol_s ? rtol_s[s] : ko->rtol) * beta[s], atol_s ? atol_s[s] : ko->atol);
    }
    PINT_CHECK(cudaMemcpyAsync(ctx->gm_tol, tol.data(), sizeof(double) * S, cudaMemcpyHostToDevice, st));
    *ctx->h_cap = ko->max_iters;  // per-slice budget, applied by the Givens update on the device
    PINT_CHECK(cudaMemcpyAsync(ctx->gm_cap, ctx->h_cap, sizeof(int), cudaMemcpyHostToDevice, st));
    // Gram-Schmidt passes per slice, from the slice's own relative tolerance:
    // one classical pass (PETSc's GMRES default) at loose tolerances -- the
    // inexact-Newton solves here run at 3e-5 .. 1e-5 relative, where CGS2
    // measured the same Krylov counts on c1-c4 at 5-9 % lower throughput --
    // and CGS2 below 1e-7 relative, where one pass loses orthogonality (a c1
    // test system at 1e-8: 41 vs 26 iterations).  PINT_CGS=1|2 forces one.
    {
      std::vector<int> two(S, 0);
      int any = 0;
      for (int s = 0; s < S; ++s) {
        two[s] = ctx->cgs_passes ? (ctx->cgs_passes == 2) : (tol[s] < 1e-7 * beta[s]);
        any |= two[s];
      }
      ctx->cur_passes = any ? 2 : 1;
      PINT_CHECK(cudaMemcpyAsync(ctx->gm_two_pass, two.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st));
    }
    std::vector<int> its(S, 0);
    std::vector<double> res(beta);
    const double* rvec = b;  // residual of the current cycle start
    PINT_CHECK(cudaMemsetAsync(ctx->gm_its, 0, sizeof(int) * S, st));
    for (int cycle = 0;; ++cycle) {
      // slices that run this cycle
      std::vector<int> cyc(S, 0);
      int ncyc = 0;
      for (int s = 0; s < S; ++s) {
        cyc[s] = host_mask[s] && res[s] > tol[s] && its[s] < ko->max_iters && std::isfinite(res[s]);
        ncyc += cyc[s];
      }
      if (ncyc == 0) break;
      PINT_CHECK(cudaMemcpyAsync(ctx->cyc_active, cyc.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st));
      PINT_CHECK(cudaMemcpyAsync(ctx->gm_active, cyc.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st));
      PINT_CHECK(cudaMemsetAsync(ctx->gm_steps, 0, sizeof(int) * S, st));
      // v0 = r / beta ; g = (beta, 0, ...)
      std::vector<double> g0((size_t)S * (m + 1), 0.0);
      for (int s = 0; s < S; ++s) g0[(size_t)s * (m + 1)] = res[s];
      PINT_CHECK(cudaMemcpyAsync(ctx->gv, g0.data(), sizeof(double) * g0.size(), cudaMemcpyHostToDevice, st));
      PINT_CHECK(cudaMemcpyAsync(ctx->gm_beta, res.data(), sizeof(double) * S, cudaMemcpyHostToDevice, st));
      pint_launch(ctx, st, k_scale_inv, vec_grid(n, S), 256, 0, ctx->V, rvec, ctx->gm_beta, n, ctx->cyc_active);
      for (int j = 0; j < m; ++j) {
        PINT_TRY(run_arnoldi(ctx, S, j, st));
        PINT_LAUNCHED();
        // poll: any slice still iterating?
        if ((j + 1) % ctx->poll_every == 0 || j + 1 == m) {
          PINT_CHECK(cudaMemcpyAsync(ctx->h_int, ctx->gm_active, sizeof(int) * S, cudaMemcpyDeviceToHost, st));
          PINT_CHECK(cudaStreamSynchronize(st));
          bool any = false;
          for (int s = 0; s < S; ++s) any = any || ctx->h_int[s];
          if (!any) break;
        }
      }
      // x += Z y  (flexible GMRES: the preconditioned directions are stored)
      pint_launch(ctx, st, k_gmres_solve, (S + 127) / 128, 128, 0, m, ctx->H, ctx->gv, ctx->gm_steps, ctx->ybuf, ctx->cyc_active,
                                                    S);
      pint_launch(ctx, st, k_mcombine, vec_grid(n, S), 256, 0, ctx->u, ctx->Z, vstride, ctx->ybuf, m + 1, ctx->gm_steps, n,
                                                 ctx->cyc_active);
      pint_launch(ctx, st, k_axpy_one, vec_grid(n, S), 256, 0, x, ctx->u, n, ctx->cyc_active);
      // true residual r = b - J x into ctx->u (reused as cycle start)
      if (ctx->matrix_free) {
        PINT_TRY(jvp(ctx, S, ctx->mf_y, ctx->mf_yo, x, ctx->u, st));
        pint_launch(ctx, st, k_bsub, vec_grid(n, S), 256, 0, ctx->u, b, n, (const int*)ctx->cyc_active);
      } else if (wide(ctx->g.nn, S))
        pint_launch(ctx, st, k_spmv<D, true, 3>, row_grid(ctx->g.nn, S), row_block<D>(), 0, ctx->g, ctx->lv[0].A, x, b, ctx->u, ctx->cyc_active);
      else
        pint_launch(ctx, st, k_spmv<D, true, 9>, row_grid(ctx->g.nn, S), row_block<D>(), 0, ctx->g, ctx->lv[0].A, x, b, ctx->u, ctx->cyc_active);
      rvec = ctx->u;
      PINT_TRY(norms(ctx, S, ctx->u, ctx->u, ctx->cyc_active, true, nullptr, nullptr, st));
      PINT_CHECK(cudaMemcpyAsync(ctx->h_dbl, ctx->d_norms, sizeof(double) * S, cudaMemcpyDeviceToHost, st));
      PINT_CHECK(cudaMemcpyAsync(ctx->h_int, ctx->gm_its, sizeof(int) * S, cudaMemcpyDeviceToHost, st));
      PINT_CHECK(cudaStreamSynchronize(st));
      for (int s = 0; s < S; ++s)
        if (cyc[s]) {
          res[s] = ctx->h_dbl[s];
          its[s] = ctx->h_int[s];
        }
    }
    for (int s = 0; s < S; ++s) {
      if (h_its) h_its[s] = its[s];
      if (h_res) h_res[s] = res[s];
    }
    return PINT_OK;
  }

  // ---- one shifted-CN step for the slices in `act` (host), Newton per slice
  //      (control flow of linalg.py:207-248)
  static int newton_step(pint_ctx* ctx, int S, int step, const double* yo, double* y, const std::vector<int>& act,
                         const pint_newton_opts* no, const pint_krylov_opts* ko, std::vector<int>& nit,
                         std::vector<int>& kit, std::vector<int>& status, cudaStream_t st) {
    const size_t n = vs(ctx);
    std::vector<double> rnorm(S), target(S), tnorm(S), lam(S, 1.0);
    std::vector<int> running(S, 0), its(S, 0), ls(S, 0), accept(S, 0);
    PINT_CHECK(cudaMemcpyAsync(ctx->d_active, act.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st));
    pint_launch(ctx, st, k_copy_active, vec_grid(n, S), 256, 0, y, yo, n, ctx->d_active);  // Newton guess = previous state
    PINT_TRY(residual(ctx, S, y, yo, ctx->r, ctx->d_active, rnorm.data(), st));
    for (int s = 0; s < S; ++s) {
      if (!act[s]) continue;
      if (!std::isfinite(rnorm[s])) { status[s] = PINT_NUMERIC_BREAKDOWN; continue; }
      target[s] = no->abs_tol + no->rel_tol * rnorm[s];
      running[s] = rnorm[s] > target[s];
    }
    std::vector<int> klin(S, 0);
    std::vector<double> kres(S, 0.0);
    for (int it = 0; it < no->max_iters; ++it) {
      int nrun = 0;
      for (int s = 0; s < S; ++s) nrun += running[s];
      if (nrun == 0) break;
      PINT_CHECK(cudaMemcpyAsync(ctx->d_active, running.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st));
      PINT_TRY(assemble(ctx, S, y, yo, ctx->d_active, st));
      // multigrid hierarchy per slice: rebuilt every Newton iteration
      // (precond_reuse = 0), or at the first Newton iteration of a step when
      // precond_reuse steps have passed since the slice's last build OR its
      // previous first-iteration solve needed more than 1.5x (+2) the Krylov
      // iterations of the first solve after that build (the operator drifted
      // away from the preconditioner).  Per-slice rule from the slice's own
      // counts, so a slice's preconditioner never depends on the batch.
      std::vector<int> built_now(S, 0);
      {
        std::vector<int> need(S, 0);
        int nneed = 0;
        for (int s = 0; s < S; ++s) {
          if (!running[s]) continue;
          const int last = ctx->built_step[s];
          const bool drift = ctx->drift_num > 0 && ctx->base_its[s] >= 0 &&
                             2 * ctx->first_its[s] > ctx->drift_num * ctx->base_its[s] + 4;
          need[s] = ko->precond_reuse <= 0 || last < 0 ||
                    (it == 0 && (step - last >= ko->precond_reuse || drift));
          if (need[s]) { ctx->built_step[s] = step; built_now[s] = it == 0; ++nneed; }
        }
        if (nneed) {
          PINT_CHECK(cudaMemcpyAsync(ctx->d_mask2, need.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st));
          PINT_TRY(precond_setup(ctx, S, ko, ctx->d_mask2, st));
        }
      }
      pint_launch(ctx, st, k_negate, vec_grid(n, S), 256, 0, ctx->b, ctx->r, n, ctx->d_active);
      // inexact Newton forcing (per slice): the first Newton iteration of a step only
      // needs rtol_first (its update error is dominated by the nonlinearity); later
      // iterations solve to rtol, but never below a tenth of the Newton target
      std::vector<double> lin_rtol(S), lin_atol(S);
      for (int s = 0; s < S; ++s) {
        lin_rtol[s] = (its[s] == 0 && ko->rtol_first > 0.0) ? std::max(ko->rtol, ko->rtol_first) : ko->rtol;
        lin_atol[s] = std::max(ko->atol, ctx->forcing * target[s]);
      }
      PINT_TRY(gmres(ctx, S, ctx->b, ctx->dx, ctx->d_active, ko, lin_rtol.data(), lin_atol.data(), klin.data(),
                     kres.data(), st, running.data(), ctx->host_beta ? rnorm.data() : nullptr));
      for (int s = 0; s < S; ++s) {
        if (!running[s]) continue;
        kit[s] += klin[s];
        if (it == 0) {
          ctx->first_its[s] = klin[s];
          if (built_now[s]) ctx->base_its[s] = klin[s];
        }
      }
      if (ctx->verbose)
        for (int s = 0; s < S; ++s)
          if (running[s])
            fprintf(stderr, "[pint] newton it %d slice %d |r| %.3e gmres its %d res %.3e\n", it, s, rnorm[s], klin[s],
                    kres[s]);
      // line search: lambda = 1, halve until decrease or damping_min (accept anyway)
      for (int s = 0; s < S; ++s) { lam[s] = 1.0; ls[s] = running[s]; }
      for (;;) {
        int nls = 0;
        for (int s = 0; s < S; ++s) nls += ls[s];
        if (nls == 0) break;
        PINT_CHECK(cudaMemcpyAsync(ctx->d_mask2, ls.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st));
        PINT_CHECK(cudaMemcpyAsync(ctx->d_lam, lam.data(), sizeof(double) * S, cudaMemcpyHostToDevice, st));
        pint_launch(ctx, st, k_trial, vec_grid(n, S), 256, 0, ctx->ytrial, y, ctx->dx, ctx->d_lam, n, ctx->d_mask2);
        std::vector<double> tn(S, 0.0);
        PINT_TRY(residual(ctx, S, ctx->ytrial, yo, ctx->rtrial, ctx->d_mask2, tn.data(), st));
        for (int s = 0; s < S; ++s) {
          if (!ls[s]) continue;
          tnorm[s] = std::isfinite(tn[s]) ? tn[s] : INFINITY;
          if (tnorm[s] < rnorm[s] || lam[s] <= no->damping_min) ls[s] = 0;
          else lam[s] = std::max(lam[s] / 2.0, no->damping_min);
        }
      }
      for (int s = 0; s < S; ++s) {
        accept[s] = 0;
        if (!running[s]) continue;
        if (!std::isfinite(tnorm[s])) {
          status[s] = PINT_NUMERIC_BREAKDOWN;
          running[s] = 0;
          continue;
        }
        accept[s] = 1;
      }
      PINT_CHECK(cudaMemcpyAsync(ctx->d_mask2, accept.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st));
      pint_launch(ctx, st, k_copy_active, vec_grid(n, S), 256, 0, y, ctx->ytrial, n, ctx->d_mask2);
      pint_launch(ctx, st, k_copy_active, vec_grid(n, S), 256, 0, ctx->r, ctx->rtrial, n, ctx->d_mask2);
      PINT_LAUNCHED();
      for (int s = 0; s < S; ++s) {
        if (!accept[s]) continue;
        rnorm[s] = tnorm[s];
        its[s] += 1;
        running[s] = rnorm[s] > target[s];
      }
    }
    for (int s = 0; s < S; ++s) {
      if (!act[s] || status[s] != PINT_OK) continue;
      nit[s] += its[s];
      if (rnorm[s] > target[s]) status[s] = PINT_NEWTON_MAX_ITERS;
    }
    return PINT_OK;
  }

  static int propagate(pint_ctx* ctx, int S, const double* y_in, double* y_out, const double* t0,
                       const double* t_end, const int* nsteps, double k, double theta0, const pint_newton_opts* no,
                       const pint_krylov_opts* ko, int* newton_iters, int* krylov_iters, int* status_out,
                       double* fail_t, cudaStream_t st) {
    const size_t n = vs(ctx);
    PINT_CHECK(cudaMemcpyAsync(ctx->ystate, y_in, sizeof(double) * n * S, cudaMemcpyDeviceToDevice, st));
    std::vector<double> t(t0, t0 + S);
    std::vector<int> nit(S, 0), kit(S, 0), status(S, PINT_OK);
    ctx->built_step.assign(ctx->maxS, -1);
    ctx->base_its.assign(ctx->maxS, -1);
    ctx->first_its.assign(ctx->maxS, 0);
    std::vector<double> ft(S, 0.0);
    int nmax = 0;
    for (int s = 0; s < S; ++s) nmax = std::max(nmax, nsteps[s]);
    std::vector<StepScalars> sts(S);
    for (int j = 0; j < nmax; ++j) {
      std::vector<int> act(S, 0);
      std::vector<double> t1(S, 0.0);
      for (int s = 0; s < S; ++s) {
        if (j >= nsteps[s] || status[s] != PINT_OK) continue;
        const double kk = (j == nsteps[s] - 1) ? (t_end[s] - t[s]) : k;
        const double theta = std::min(std::max(0.5 + theta0 * kk, 0.5), 1.0);
        t1[s] = t[s] + kk;
        sts[s] = make_step(ctx->desc, kk, theta, t1[s]);
        act[s] = 1;
      }
      PINT_CHECK(cudaMemcpyAsync(ctx->d_st, sts.data(), sizeof(StepScalars) * S, cudaMemcpyHostToDevice, st));
      PINT_TRY(newton_step(ctx, S, j, ctx->ystate, ctx->ynew, act, no, ko, nit, kit, status, st));
      std::vector<int> ok(S, 0);
      for (int s = 0; s < S; ++s) {
        if (!act[s]) continue;
        if (status[s] != PINT_OK) { ft[s] = t1[s]; continue; }
        ok[s] = 1;
        t[s] = t1[s];
      }
      PINT_CHECK(cudaMemcpyAsync(ctx->d_mask2, ok.data(), sizeof(int) * S, cudaMemcpyHostToDevice, st));
      pint_launch(ctx, st, k_copy_active, vec_grid(n, S), 256, 0, ctx->ystate, ctx->ynew, n, ctx->d_mask2);
      PINT_LAUNCHED();
    }
    PINT_CHECK(cudaMemcpyAsync(y_out, ctx->ystate, sizeof(double) * n * S, cudaMemcpyDeviceToDevice, st));
    PINT_CHECK(cudaStreamSynchronize(st));
    for (int s = 0; s < S; ++s) {
      if (newton_iters) newton_iters[s] = nit[s];
      if (krylov_iters) krylov_iters[s] = kit[s];
      if (status_out) status_out[s] = status[s];
      if (fail_t) fail_t[s] = ft[s];
    }
    return PINT_OK;
  }

  // ================================================================ device-driven control flow
  // The whole propagate call captured as ONE CUDA graph whose WHILE / IF
  // conditional nodes are driven by the controller kernels of
  // kernels_loop.cuh: time steps -> Newton iterations -> (multigrid rebuild)
  // -> GMRES cycles -> Arnoldi steps, and the line search.  The control flow is
  // the host path's (propagate / newton_step / gmres above) statement for
  // statement; every per-slice decision is made on the device from the
  // slice's own numbers, so there is no host round trip inside the call and the
  // result equals the host-driven path bitwise.
  // one restart cycle of flexible GMRES(m) on stream s (depth dp): v0 = u / beta,
  // the Arnoldi steps (the first ctx->gate0 unconditionally, the rest under
  // IF(any slice still iterating) in blocks of ctx->gate), the update
  // x += Z y, the true residual u = b - J x and its norm; two: the second
  // Gram-Schmidt pass runs (masked per slice)
  static int capture_cycle(pint_ctx* ctx, int S, bool two, cudaStream_t s3, int dp3) {
    const size_t n = vs(ctx);
    const int m = ctx->restart;
    const size_t vstride = (size_t)ctx->maxS * n;
    const LoopDev d = ctx->ld;
    pint_launch(ctx, s3, k_scale_inv, vec_grid(n, S), 256, 0, ctx->V, (const double*)ctx->u,
                (const double*)ctx->gm_beta, n, (const int*)ctx->cyc_active);
    const int j_free = std::min(m, ctx->gate0);
    for (int j = 0; j < j_free; ++j) PINT_TRY(arnoldi_step_dev(ctx, S, j, two, s3));
    for (int j0 = j_free; j0 < m; j0 += ctx->gate) {
      const int j1 = std::min(m, j0 + ctx->gate);
      cudaGraphConditionalHandle h_j;
      const int i_j = (int)ctx->body_nodes.size();
      PINT_TRY(new_cond(ctx, &h_j));
      pint_launch(ctx, s3, k_arnoldi_gate, 1, kLoopThreads, 0, d, h_j, i_j);
      PINT_TRY(capture_cond(ctx, s3, dp3, h_j, false, i_j, [&](cudaStream_t s4, int) -> int {
        for (int j = j0; j < j1; ++j) PINT_TRY(arnoldi_step_dev(ctx, S, j, two, s4));
        return PINT_OK;
      }));
    }
    pint_launch(ctx, s3, k_gmres_solve, (S + 127) / 128, 128, 0, m, (const double*)ctx->H, (const double*)ctx->gv,
                (const int*)ctx->gm_steps, ctx->ybuf, (const int*)ctx->cyc_active, S);
    pint_launch(ctx, s3, k_mcombine, vec_grid(n, S), 256, 0, ctx->u, (const double*)ctx->Z, vstride,
                (const double*)ctx->ybuf, m + 1, (const int*)ctx->gm_steps, n, (const int*)ctx->cyc_active);
    pint_launch(ctx, s3, k_axpy_one, vec_grid(n, S), 256, 0, ctx->dx, (const double*)ctx->u, n,
                (const int*)ctx->cyc_active);
    if (wide(ctx->g.nn, S))
      pint_launch(ctx, s3, k_spmv<D, true, 3>, row_grid(ctx->g.nn, S), row_block<D>(), 0, ctx->g,
                  (const double*)ctx->lv[0].A, (const double*)ctx->dx, (const double*)ctx->b, ctx->u,
                  (const int*)ctx->cyc_active);
    else
      pint_launch(ctx, s3, k_spmv<D, true, 9>, row_grid(ctx->g.nn, S), row_block<D>(), 0, ctx->g,
                  (const double*)ctx->lv[0].A, (const double*)ctx->dx, (const double*)ctx->b, ctx->u,
                  (const int*)ctx->cyc_active);
    return norms(ctx, S, ctx->u, ctx->u, ctx->cyc_active, true, nullptr, nullptr, s3);
  }

  // one line-search trial: y_trial = y + lambda dx, its residual norm, the
  // halving rule (linalg.py:226-237); sets the line-search handle
  static int capture_trial(pint_ctx* ctx, int S, cudaGraphConditionalHandle h_ls, int i_ls, cudaStream_t st) {
    const size_t n = vs(ctx);
    const LoopDev d = ctx->ld;
    pint_launch(ctx, st, k_trial, vec_grid(n, S), 256, 0, ctx->ytrial, (const double*)ctx->ynew,
                (const double*)ctx->dx, (const double*)d.lam, n, (const int*)d.ls_mask);
    PINT_TRY(residual(ctx, S, ctx->ytrial, ctx->ystate, ctx->rtrial, d.ls_mask, nullptr, st));
    pint_launch(ctx, st, k_ls_update, 1, kLoopThreads, 0, d, h_ls, i_ls);
    return PINT_OK;
  }

  // one Newton iteration (linalg.py:220-240); sets the Newton handle
  static int capture_newton_iter(pint_ctx* ctx, int S, const pint_krylov_opts* ko, cudaGraphConditionalHandle h_newton,
                                 int i_newton, cudaStream_t s2, int dp2) {
    const size_t n = vs(ctx);
    const LoopDev d = ctx->ld;
    PINT_TRY(assemble(ctx, S, ctx->ynew, ctx->ystate, d.running, s2));
    cudaGraphConditionalHandle h_prec;
    const int i_prec = (int)ctx->body_nodes.size();
    PINT_TRY(new_cond(ctx, &h_prec));
    pint_launch(ctx, s2, k_precond_decide, 1, kLoopThreads, 0, d, h_prec, i_prec);
    PINT_TRY(capture_cond(ctx, s2, dp2, h_prec, false, i_prec, [&](cudaStream_t s3, int) -> int {
      return precond_setup(ctx, S, ko, d.need, s3);
    }));
    pint_launch(ctx, s2, k_gmres_prep, vec_grid(n, S), 256, 0, ctx->b, ctx->dx, ctx->u, (const double*)ctx->r, n,
                (const int*)d.running);
    // restart cycles: two-pass loop first (a solve can only drop from two passes to one)
    cudaGraphConditionalHandle h1, h2;
    const int i1 = (int)ctx->body_nodes.size();
    PINT_TRY(new_cond(ctx, &h1));
    const int i2 = (int)ctx->body_nodes.size();
    PINT_TRY(new_cond(ctx, &h2));
    pint_launch(ctx, s2, k_gmres_init, 1, kLoopThreads, 0, d, h1, i1, h2, i2);
    for (int two = 1; two >= 0; --two)
      PINT_TRY(capture_cond(ctx, s2, dp2, two ? h2 : h1, true, two ? i2 : i1, [&](cudaStream_t s3, int dp3) -> int {
        PINT_TRY(capture_cycle(ctx, S, two == 1, s3, dp3));
        pint_launch(ctx, s3, k_cycle_end, 1, kLoopThreads, 0, d, h1, i1, h2, i2);
        return PINT_OK;
      }));
    pint_launch(ctx, s2, k_gmres_end, 1, kLoopThreads, 0, d);
    // line search: the first trial always, further halvings under WHILE
    cudaGraphConditionalHandle h_ls;
    const int i_ls = (int)ctx->body_nodes.size();
    PINT_TRY(new_cond(ctx, &h_ls));
    PINT_TRY(capture_trial(ctx, S, h_ls, i_ls, s2));
    PINT_TRY(capture_cond(ctx, s2, dp2, h_ls, true, i_ls, [&](cudaStream_t s3, int) -> int {
      return capture_trial(ctx, S, h_ls, i_ls, s3);
    }));
    pint_launch(ctx, s2, k_accept_copy, vec_grid(n, S), 256, 0, ctx->ynew, (const double*)ctx->ytrial, ctx->r,
                (const double*)ctx->rtrial, n, (const int*)d.running, (const double*)d.tnorm);
    pint_launch(ctx, s2, k_newton_update, 1, kLoopThreads, 0, d, h_newton, i_newton);
    PINT_LAUNCHED();
    return PINT_OK;
  }

  static int capture_propagate(pint_ctx* ctx, int S, const pint_krylov_opts* ko, cudaStream_t st0) {
    const size_t n = vs(ctx);
    const LoopDev d = ctx->ld;
    cudaGraphConditionalHandle h_step;
    const int i_step = (int)ctx->body_nodes.size();
    PINT_TRY(new_cond(ctx, &h_step));
    pint_launch(ctx, st0, k_loop_init, 1, kLoopThreads, 0, d, h_step, i_step);
    return capture_cond(ctx, st0, 0, h_step, true, i_step, [&](cudaStream_t s1, int dp1) -> int {
      // ---- one time step (integrators.py:154-162; guess = previous state, integrators.py:93)
      pint_launch(ctx, s1, k_step_begin, 1, kLoopThreads, 0, d);
      pint_launch(ctx, s1, k_copy_active, vec_grid(n, S), 256, 0, ctx->ynew, (const double*)ctx->ystate, n,
                  (const int*)d.act);
      PINT_TRY(residual(ctx, S, ctx->ynew, ctx->ystate, ctx->r, d.act, nullptr, s1));
      cudaGraphConditionalHandle h_newton;
      const int i_newton = (int)ctx->body_nodes.size();
      PINT_TRY(new_cond(ctx, &h_newton));
      pint_launch(ctx, s1, k_newton_init, 1, kLoopThreads, 0, d, h_newton, i_newton);
      // the first Newton iteration always (a converged start runs it masked), the rest under WHILE
      PINT_TRY(capture_newton_iter(ctx, S, ko, h_newton, i_newton, s1, dp1));
      PINT_TRY(capture_cond(ctx, s1, dp1, h_newton, true, i_newton, [&](cudaStream_t s2, int dp2) -> int {
        return capture_newton_iter(ctx, S, ko, h_newton, i_newton, s2, dp2);
      }));
      pint_launch(ctx, s1, k_step_end, 1, kLoopThreads, 0, d, h_step, i_step);
      pint_launch(ctx, s1, k_copy_active, vec_grid(n, S), 256, 0, ctx->ystate, (const double*)ctx->ynew, n,
                  (const int*)d.ok);
      PINT_LAUNCHED();
      return PINT_OK;
    });
  }
};

// Public calls run on the context's own non-blocking stream (so Arnoldi
// steps can be graph-captured), ordered after / before the caller's stream.
struct StreamGuard {
  pint_ctx* ctx;
  cudaStream_t user;
  StreamGuard(pint_ctx* c, void* s) : ctx(c), user((cudaStream_t)s) {
    cudaEventRecord(ctx->ev_in, user);
    cudaStreamWaitEvent(ctx->stream, ctx->ev_in, 0);
  }
  ~StreamGuard() {
    cudaEventRecord(ctx->ev_out, ctx->stream);
    cudaStreamWaitEvent(user, ctx->ev_out, 0);
  }
};

int upload_steps(pint_ctx* ctx, int S, const double* k, const double* theta, const double* t1, cudaStream_t st) {
  std::vector<StepScalars> sts(S);
  for (int s = 0; s < S; ++s) sts[s] = make_step(ctx->desc, k[s], theta[s], t1[s]);
  PINT_CHECK(cudaMemcpyAsync(ctx->d_st, sts.data(), sizeof(StepScalars) * S, cudaMemcpyHostToDevice, st));
  return PINT_OK;
}

int check_S(pint_ctx* ctx, int S) {
  if (!ctx) return PINT_INVALID_ARG;
  if (S < 1 || S > ctx->maxS) {
    ctx->err = "batch size " + std::to_string(S) + " outside [1, " + std::to_string(ctx->maxS) + "]";
    return PINT_INVALID_ARG;
  }
  return PINT_OK;
}

// ---------------------------------------------------------------- device-driven propagate (host side)
int mf_reject(pint_ctx* ctx, const char* what) {
  ctx->err = std::string(what) + " needs the Jacobian / multigrid hierarchy, which a matrix-free context "
                                 "(PINT_CTX_MATRIX_FREE) does not hold";
  return PINT_INVALID_ARG;
}

// the device-driven loop covers every option except the diagnostics that need
// the host in the loop (per-iteration trace, CUDA-event profiling) and the
// A/B variants kept for measurement (split norm, fused Arnoldi kernel)
bool use_device_loop(const pint_ctx* ctx) {
  return ctx->device_loop && !ctx->prof && !ctx->verbose && !ctx->split_norm && !ctx->use_fused;
}

template <typename T>
int grow(pint_ctx* ctx, T** d, T** h, size_t count) {
  if (*d) cudaFree(*d);
  if (h && *h) cudaFreeHost(*h);
  *d = nullptr;
  if (h) *h = nullptr;
  PINT_CHECK(cudaMalloc((void**)d, sizeof(T) * std::max<size_t>(count, 1)));
  if (h) PINT_CHECK(cudaMallocHost((void**)h, sizeof(T) * std::max<size_t>(count, 1)));
  return PINT_OK;
}

// step tables for `entries` (step, slice) pairs and call scalars for `slots` slices
int ensure_tables(pint_ctx* ctx, size_t entries, size_t slots) {
  if (entries > ctx->tab_cap) {
    const size_t cap = std::max(entries, 2 * ctx->tab_cap);
    PINT_TRY(grow(ctx, &ctx->d_sts, &ctx->h_sts, cap));
    PINT_TRY(grow(ctx, &ctx->d_t1tab, &ctx->h_t1tab, cap));
    ctx->tab_cap = cap;
  }
  if (slots > ctx->lsv_cap) {
    const size_t cap = std::max(slots, 2 * ctx->lsv_cap);
    PINT_TRY(grow(ctx, &ctx->d_nsteps, &ctx->h_nsteps, cap));
    PINT_TRY(grow(ctx, &ctx->d_lsv, &ctx->h_lsv, cap));
    ctx->lsv_cap = cap;
  }
  return PINT_OK;
}

// steps of slice s into the tables at column s of a [nmax][S] block starting
// at `off`: the time arithmetic of Impl::propagate (integrators.py:154-162)
void fill_steps(pint_ctx* ctx, size_t off, int S, int s, int nsteps, int nmax, double t0, double t_end, double k,
                double theta0) {
  double t = t0;
  for (int j = 0; j < nmax; ++j) {
    const size_t e = off + (size_t)j * S + s;
    if (j >= nsteps) {
      ctx->h_sts[e] = StepScalars{};
      ctx->h_t1tab[e] = 0.0;
      continue;
    }
    const double kk = (j == nsteps - 1) ? (t_end - t) : k;
    const double theta = std::min(std::max(0.5 + theta0 * kk, 0.5), 1.0);
    const double t1 = t + kk;
    ctx->h_sts[e] = make_step(ctx->desc, kk, theta, t1);
    ctx->h_t1tab[e] = t1;
    t = t1;
  }
}

LoopScalars call_scalars(pint_ctx* ctx, int S, int nmax, const pint_newton_opts* no, const pint_krylov_opts* ko,
                         size_t tab_off, size_t nsteps_off) {
  LoopScalars L{};
  L.S = S;
  L.nmax = nmax;
  L.m = ctx->restart;
  L.newton_max = no->max_iters;
  L.lin_max = ko->max_iters;
  L.reuse = ko->precond_reuse;
  L.drift_num = ctx->drift_num;
  L.cgs_force = ctx->cgs_passes;
  L.abs_tol = no->abs_tol;
  L.rel_tol = no->rel_tol;
  L.damping_min = no->damping_min;
  L.lin_rtol = ko->rtol;
  L.lin_rtol_first = ko->rtol_first;
  L.lin_atol = ko->atol;
  L.forcing = ctx->forcing;
  L.sts = ctx->d_sts + tab_off;
  L.t1tab = ctx->d_t1tab + tab_off;
  L.nsteps = ctx->d_nsteps + nsteps_off;
  return L;
}

int get_loop_graph(pint_ctx* ctx, int S, const pint_krylov_opts* ko, cudaStream_t st,
                   std::pair<cudaGraphExec_t, long long>** out) {
  const std::vector<double> key = {(double)S, (double)ko->pre_smooth, (double)ko->post_smooth, ko->omega,
                                   (double)ko->max_levels, (double)ko->coarse_sweeps, (double)ko->smoother};
  auto it = ctx->loop_graphs.find(key);
  if (it == ctx->loop_graphs.end()) {
    const size_t bodies0 = ctx->body_nodes.size();
    const long long before = ctx->launches;
    ctx->capturing = true;
    ctx->nopdl.clear();
    cudaGraph_t graph = nullptr;
    int rc = PINT_OK;
    cudaError_t e = cudaStreamBeginCapture(st, cudaStreamCaptureModeRelaxed);
    if (e == cudaSuccess) {
      cudaStreamCaptureStatus cs;
      e = cudaStreamGetCaptureInfo(st, &cs, nullptr, &ctx->cap_root, nullptr, nullptr);
      if (e == cudaSuccess)
        rc = ctx->D == 2 ? Impl<2>::capture_propagate(ctx, S, ko, st) : Impl<3>::capture_propagate(ctx, S, ko, st);
      const cudaError_t e2 = cudaStreamEndCapture(st, &graph);
      if (e == cudaSuccess) e = e2;
    }
    ctx->capturing = false;
    ctx->nopdl.clear();
    const long long top = ctx->launches - before;
    ctx->launches = before;
    if (rc == PINT_OK && e != cudaSuccess) {
      ctx->err = std::string("loop-graph capture: ") + cudaGetErrorString(e);
      rc = PINT_CUDA_ERROR;
    }
    cudaGraphExec_t exec = nullptr;
    if (rc == PINT_OK) {
      e = cudaGraphInstantiate(&exec, graph, 0);
      if (e != cudaSuccess) {
        ctx->err = std::string("loop-graph instantiate: ") + cudaGetErrorString(e);
        rc = PINT_CUDA_ERROR;
      }
    }
    if (graph) cudaGraphDestroy(graph);
    if (rc != PINT_OK) {
      ctx->body_nodes.resize(bodies0);
      cudaGetLastError();
      return rc;
    }
    PINT_CHECK(cudaMemcpy(ctx->d_body_nodes + bodies0, ctx->body_nodes.data() + bodies0,
                          sizeof(int) * (ctx->body_nodes.size() - bodies0), cudaMemcpyHostToDevice));
    it = ctx->loop_graphs.emplace(key, std::make_pair(exec, top)).first;
  }
  *out = &it->second;
  return PINT_OK;
}

int propagate_dev(pint_ctx* ctx, int S, const double* y_in, double* y_out, const double* t0, const double* t_end,
                  const int* nsteps, double k, double theta0, const pint_newton_opts* no,
                  const pint_krylov_opts* ko, int* newton_iters, int* krylov_iters, int* status_out, double* fail_t,
                  cudaStream_t st) {
  const size_t n = (size_t)ctx->C * ctx->g.np;
  int nmax = 0;
  for (int s = 0; s < S; ++s) nmax = std::max(nmax, (int)nsteps[s]);
  PINT_TRY(ensure_tables(ctx, (size_t)std::max(nmax, 1) * S, S));
  for (int s = 0; s < S; ++s) {
    fill_steps(ctx, 0, S, s, nsteps[s], nmax, t0[s], t_end[s], k, theta0);
    ctx->h_nsteps[s] = nsteps[s];
  }
  *ctx->h_ls = call_scalars(ctx, S, nmax, no, ko, 0, 0);
  std::pair<cudaGraphExec_t, long long>* graph = nullptr;
  PINT_TRY(get_loop_graph(ctx, S, ko, st, &graph));
  const size_t ents = (size_t)std::max(nmax, 1) * S;
  PINT_CHECK(cudaMemcpyAsync(ctx->d_sts, ctx->h_sts, sizeof(StepScalars) * ents, cudaMemcpyHostToDevice, st));
  PINT_CHECK(cudaMemcpyAsync(ctx->d_t1tab, ctx->h_t1tab, sizeof(double) * ents, cudaMemcpyHostToDevice, st));
  PINT_CHECK(cudaMemcpyAsync(ctx->d_nsteps, ctx->h_nsteps, sizeof(int) * S, cudaMemcpyHostToDevice, st));
  PINT_CHECK(cudaMemcpyAsync(ctx->ld.ls, ctx->h_ls, sizeof(LoopScalars), cudaMemcpyHostToDevice, st));
  PINT_CHECK(cudaMemcpyAsync(ctx->ystate, y_in, sizeof(double) * n * S, cudaMemcpyDeviceToDevice, st));
  PINT_CHECK(cudaGraphLaunch(graph->first, st));
  ctx->launches += graph->second;
  PINT_CHECK(cudaMemcpyAsync(y_out, ctx->ystate, sizeof(double) * n * S, cudaMemcpyDeviceToDevice, st));
  int* hi = ctx->h_out_i;
  PINT_CHECK(cudaMemcpyAsync(hi, ctx->ld.status, sizeof(int) * S, cudaMemcpyDeviceToHost, st));
  PINT_CHECK(cudaMemcpyAsync(hi + ctx->maxS, ctx->ld.nit, sizeof(int) * S, cudaMemcpyDeviceToHost, st));
  PINT_CHECK(cudaMemcpyAsync(hi + 2 * ctx->maxS, ctx->ld.kit, sizeof(int) * S, cudaMemcpyDeviceToHost, st));
  PINT_CHECK(cudaMemcpyAsync(ctx->h_out_d, ctx->ld.ft, sizeof(double) * S, cudaMemcpyDeviceToHost, st));
  PINT_CHECK(cudaStreamSynchronize(st));
  for (int s = 0; s < S; ++s) {
    if (status_out) status_out[s] = hi[s];
    if (newton_iters) newton_iters[s] = hi[ctx->maxS + s];
    if (krylov_iters) krylov_iters[s] = hi[2 * ctx->maxS + s];
    if (fail_t) fail_t[s] = ctx->h_out_d[s];
  }
  return PINT_OK;
}

int ensure_sweep(pint_ctx* ctx, size_t L) {
  if (L <= ctx->sw_cap) return PINT_OK;
  const size_t cap = std::max(L, 2 * ctx->sw_cap);
  const int nblk = (ctx->g.np + kRedChunk - 1) / kRedChunk;
  const size_t part = std::max((size_t)ctx->C * 5 * nblk, cap * 2 * (size_t)ctx->nblk);
  PINT_TRY(grow<double>(ctx, &ctx->sw_part, nullptr, part));
  PINT_TRY(grow<double>(ctx, &ctx->sw_theta, nullptr, cap));
  PINT_TRY(grow<double>(ctx, &ctx->sw_corr, nullptr, cap));
  PINT_TRY(grow<double>(ctx, &ctx->sw_ft, nullptr, cap));
  PINT_TRY(grow<int>(ctx, &ctx->sw_status, nullptr, cap));
  PINT_TRY(grow<int>(ctx, &ctx->sw_nit, nullptr, cap));
  PINT_TRY(grow<int>(ctx, &ctx->sw_kit, nullptr, cap));
  if (ctx->h_sw) cudaFreeHost(ctx->h_sw);
  PINT_CHECK(cudaMallocHost((void**)&ctx->h_sw, sizeof(double) * 7 * cap));
  ctx->sw_cap = cap;
  return PINT_OK;
}

// K8b for one slice on the context's scratch: theta_l, x_new, corr_l on the device
void correct_dev(pint_ctx* ctx, int l, const double* c_new, const double* f_old, const double* c_old,
                 const double* x_prev, double* x_new, int variant, double lo, double hi, cudaStream_t st) {
  const int C = ctx->C, nn = ctx->g.nn, np = ctx->g.np;
  const int nblk = (nn + kRedChunk - 1) / kRedChunk;
  double* part3 = ctx->sw_part;
  double* part2 = ctx->sw_part + (size_t)C * 3 * nblk;
  pint_launch(ctx, st, k_block_dots, dim3(nblk, C), kRedThreads, 0, f_old, c_new, nn, np, part3, nblk);
  pint_launch(ctx, st, k_theta, 1, 32, 0, (const double*)part3, nblk, C, variant, lo, hi, ctx->sw_theta + l);
  pint_launch(ctx, st, k_update_norms, dim3(nblk, C), kRedThreads, 0, c_new, f_old, c_old, x_prev, x_new,
              (const double*)(ctx->sw_theta + l), nn, np, part2, nblk);
  pint_launch(ctx, st, k_corr, 1, 32, 0, (const double*)part2, nblk, C, ctx->sw_corr + l);
}

// the sequential corrector sweep (parareal.py:422-436) or the coarse
// initialisation (parareal.py:410-416): L loop-graph launches of batch 1 and
// the K8b kernels, all enqueued without a host synchronisation
int coarse_sweep(pint_ctx* ctx, int L, double* x, const double* x_prev, double* c_new, const double* c_old,
                 const double* f_old, const double* t_grid, const int* nsteps, double k, double theta0,
                 const pint_newton_opts* no, const pint_krylov_opts* ko, int variant, double lo, double hi,
                 double* theta_out, double* corr_out, int* newton_iters, int* krylov_iters, int* status_out,
                 double* fail_t, cudaStream_t st) {
  const size_t n = (size_t)ctx->C * ctx->g.np;
  size_t ents = 0;
  std::vector<size_t> off(L);
  for (int l = 0; l < L; ++l) {
    off[l] = ents;
    ents += (size_t)std::max(nsteps[l], 1);
  }
  PINT_TRY(ensure_tables(ctx, ents, L));
  PINT_TRY(ensure_sweep(ctx, L));
  for (int l = 0; l < L; ++l) {
    fill_steps(ctx, off[l], 1, 0, nsteps[l], std::max(nsteps[l], 1), t_grid[l], t_grid[l + 1], k, theta0);
    ctx->h_nsteps[l] = nsteps[l];
    ctx->h_lsv[l] = call_scalars(ctx, 1, nsteps[l], no, ko, off[l], l);
  }
  // host-driven fallback (PINT_DEVICE_LOOP=0 / profiling): batch-1 host loop per slice, same bits
  const bool dev_loop = use_device_loop(ctx);
  std::pair<cudaGraphExec_t, long long>* graph = nullptr;
  if (dev_loop) PINT_TRY(get_loop_graph(ctx, 1, ko, st, &graph));
  PINT_CHECK(cudaMemcpyAsync(ctx->d_sts, ctx->h_sts, sizeof(StepScalars) * ents, cudaMemcpyHostToDevice, st));
  PINT_CHECK(cudaMemcpyAsync(ctx->d_t1tab, ctx->h_t1tab, sizeof(double) * ents, cudaMemcpyHostToDevice, st));
  PINT_CHECK(cudaMemcpyAsync(ctx->d_nsteps, ctx->h_nsteps, sizeof(int) * L, cudaMemcpyHostToDevice, st));
  PINT_CHECK(cudaMemcpyAsync(ctx->d_lsv, ctx->h_lsv, sizeof(LoopScalars) * L, cudaMemcpyHostToDevice, st));
  std::vector<int> h_status(L, 0), h_nit(L, 0), h_kit(L, 0);
  std::vector<double> h_ft(L, 0.0);
  for (int l = 0; l < L; ++l) {
    double* cn = c_new + l * n;
    if (dev_loop) {
      PINT_CHECK(cudaMemcpyAsync(ctx->ystate, x + l * n, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
      PINT_CHECK(cudaMemcpyAsync(ctx->ld.ls, ctx->d_lsv + l, sizeof(LoopScalars), cudaMemcpyDeviceToDevice, st));
      PINT_CHECK(cudaGraphLaunch(graph->first, st));
      ctx->launches += graph->second;
      pint_launch(ctx, st, k_sweep_record, 1, 32, 0, ctx->ld, l, ctx->sw_status, ctx->sw_nit, ctx->sw_kit,
                  ctx->sw_ft);
    } else {
      const double t0 = t_grid[l], t1 = t_grid[l + 1];
      const int ns = nsteps[l];
      PINT_TRY(ctx->D == 2 ? Impl<2>::propagate(ctx, 1, x + l * n, cn, &t0, &t1, &ns, k, theta0, no, ko,
                                                &h_nit[l], &h_kit[l], &h_status[l], &h_ft[l], st)
                           : Impl<3>::propagate(ctx, 1, x + l * n, cn, &t0, &t1, &ns, k, theta0, no, ko,
                                                &h_nit[l], &h_kit[l], &h_status[l], &h_ft[l], st));
    }
    PINT_CHECK(cudaMemcpyAsync(cn, ctx->ystate, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
    if (f_old)
      correct_dev(ctx, l, cn, f_old + l * n, c_old + l * n, x_prev + (l + 1) * n, x + (l + 1) * n, variant, lo, hi,
                  st);
    else
      PINT_CHECK(cudaMemcpyAsync(x + (l + 1) * n, ctx->ystate, sizeof(double) * n, cudaMemcpyDeviceToDevice, st));
  }
  PINT_LAUNCHED();
  double* h = ctx->h_sw;
  const size_t cap = ctx->sw_cap;
  if (f_old) {
    PINT_CHECK(cudaMemcpyAsync(h, ctx->sw_theta, sizeof(double) * L, cudaMemcpyDeviceToHost, st));
    PINT_CHECK(cudaMemcpyAsync(h + cap, ctx->sw_corr, sizeof(double) * L, cudaMemcpyDeviceToHost, st));
  }
  PINT_CHECK(cudaMemcpyAsync(h + 2 * cap, ctx->sw_ft, sizeof(double) * L, cudaMemcpyDeviceToHost, st));
  int* hn = reinterpret_cast<int*>(h + 3 * cap);
  PINT_CHECK(cudaMemcpyAsync(hn, ctx->sw_status, sizeof(int) * L, cudaMemcpyDeviceToHost, st));
  PINT_CHECK(cudaMemcpyAsync(hn + cap, ctx->sw_nit, sizeof(int) * L, cudaMemcpyDeviceToHost, st));
  PINT_CHECK(cudaMemcpyAsync(hn + 2 * cap, ctx->sw_kit, sizeof(int) * L, cudaMemcpyDeviceToHost, st));
  PINT_CHECK(cudaStreamSynchronize(st));
  for (int l = 0; l < L; ++l) {
    if (theta_out) theta_out[l] = f_old ? h[l] : 1.0;
    if (corr_out) corr_out[l] = f_old ? h[cap + l] : 0.0;
    if (fail_t) fail_t[l] = dev_loop ? h[2 * cap + l] : h_ft[l];
    if (status_out) status_out[l] = dev_loop ? hn[l] : h_status[l];
    if (newton_iters) newton_iters[l] = dev_loop ? hn[cap + l] : h_nit[l];
    if (krylov_iters) krylov_iters[l] = dev_loop ? hn[2 * cap + l] : h_kit[l];
  }
  return PINT_OK;
}

}  // namespace

// ======================================================================== C ABI

extern "C" {

int pint_create(const pint_problem_desc* desc, int32_t max_slices, int32_t restart, pint_ctx** out) {
  return pint_create_ex(desc, max_slices, restart, 0, out);
}

int pint_create_ex(const pint_problem_desc* desc, int32_t max_slices, int32_t restart, int32_t flags,
                   pint_ctx** out) {
  if (!desc || !out || max_slices < 1 || restart < 1 || restart + 1 > kMdotMax) return PINT_INVALID_ARG;
  if (flags & ~PINT_CTX_MATRIX_FREE) return PINT_INVALID_ARG;
  if (desc->dim != 2 && desc->dim != 3) return PINT_INVALID_ARG;
  for (int m = 0; m < desc->dim; ++m)
    if (desc->cells[m] < 1) return PINT_INVALID_ARG;
  pint_ctx* ctx = new pint_ctx();
  *out = ctx;
  ctx->desc = *desc;
  ctx->D = desc->dim;
  ctx->C = 2 * desc->dim + 1;
  ctx->maxS = max_slices;
  ctx->restart = restart;
  ctx->matrix_free = (flags & PINT_CTX_MATRIX_FREE) != 0;
  ctx->verbose = std::getenv("PINT_VERBOSE") && std::getenv("PINT_VERBOSE")[0] == '1';
  ctx->use_graphs = !(std::getenv("PINT_GRAPHS") && std::getenv("PINT_GRAPHS")[0] == '0');
  ctx->use_tail = !(std::getenv("PINT_TAIL") && std::getenv("PINT_TAIL")[0] == '0');
  ctx->tail_cluster = !(std::getenv("PINT_TAIL_CLUSTER") && std::getenv("PINT_TAIL_CLUSTER")[0] == '0');
  if (const char* e = std::getenv("PINT_TAIL_CL")) {
    const int v = std::atoi(e);
    ctx->tail_cl_force = (v == 2 || v == 4 || v == 8) ? v : 0;
  }
  {
    int dev = 0, sms = 0;
    if (cudaGetDevice(&dev) == cudaSuccess &&
        cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev) == cudaSuccess && sms > 0)
      ctx->num_sms = sms;
  }
  ctx->use_fused = std::getenv("PINT_FUSED") && std::getenv("PINT_FUSED")[0] == '1';
  ctx->jac_columns = std::getenv("PINT_JAC") && std::string(std::getenv("PINT_JAC")) == "columns";
  ctx->jac_strip = !(std::getenv("PINT_JAC") && std::string(std::getenv("PINT_JAC")) == "colour");
  // tiled K1 / K2' in 2-d (c3: residual 0.52 -> 0.45 ms, J w 0.58 -> 0.56 ms); the 3-d tile spills
  // (255 registers) and measured slower (c4 residual 0.23 -> 0.25 ms), so 3-d keeps the per-point kernels
  ctx->elem_old = ctx->D == 3;
  if (const char* e = std::getenv("PINT_ELEM")) ctx->elem_old = std::string(e) == "old";
  // dynamic shared memory of the tiled element kernels (3-d J w exceeds the 48 KB default)
  cudaFuncSetAttribute(k_elem_tile<2, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ElemTile<2>::smem(2));
  cudaFuncSetAttribute(k_elem_tile<2, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ElemTile<2>::smem(3));
  cudaFuncSetAttribute(k_elem_tile<3, 0>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ElemTile<3>::smem(2));
  cudaFuncSetAttribute(k_elem_tile<3, 1>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)ElemTile<3>::smem(3));
  ctx->vanka_smem = std::getenv("PINT_VANKA_SETUP") && std::string(std::getenv("PINT_VANKA_SETUP")) == "smem";
  // level-0 Vanka sweep: fused (cell solves + gather, k_vanka_apply) in 2-d,
  // split in 3-d, where the fused grid is 1.2 waves of (node, comp) threads
  // (c4: fused 86.6 us vs split 82.9 + gather per sweep; c3: fused 212 vs 261)
  if (const char* e = std::getenv("PINT_CGS")) ctx->cgs_passes = std::atoi(e) == 2 ? 2 : 1;
  if (const char* e = std::getenv("PINT_SCALE_FUSE")) ctx->scale_fuse_max = std::atoi(e);
  ctx->defer_scale = !(std::getenv("PINT_DEFER_SCALE") && std::getenv("PINT_DEFER_SCALE")[0] == '0');
  ctx->host_beta = !(std::getenv("PINT_HOST_BETA") && std::getenv("PINT_HOST_BETA")[0] == '0');
  ctx->split_norm = std::getenv("PINT_SPLIT_NORM") && std::getenv("PINT_SPLIT_NORM")[0] == '1';
  ctx->vanka_split = ctx->D == 3;
  // default since round 2: the sweep in block-stencil form (k_vanka_stencil_apply) on every standalone
  // level; PINT_VANKA=fused|split select the cell-inverse kernels (the tail always uses cell inverses)
  ctx->vanka_stencil = true;
  if (const char* e = std::getenv("PINT_VANKA")) {
    ctx->vanka_split = std::string(e) == "split";
    ctx->vanka_stencil = std::string(e) == "stencil";
  }
  if (const char* e = std::getenv("PINT_DRIFT")) ctx->drift_num = std::atoi(e);
  if (const char* e = std::getenv("PINT_TAIL_ROWS")) ctx->tail_rows = std::atoi(e);
  ctx->pdl = !(std::getenv("PINT_PDL") && std::getenv("PINT_PDL")[0] == '0');
  ctx->spmv32_node = !(std::getenv("PINT_SPMV32") && std::string(std::getenv("PINT_SPMV32")) == "row");
  ctx->spmv32_staged = !std::getenv("PINT_SPMV32") || std::string(std::getenv("PINT_SPMV32")) == "staged";
  if (const char* e = std::getenv("PINT_SPMV32_MIN")) ctx->spmv32_min = (size_t)std::atoll(e);
  if (const char* e = std::getenv("PINT_STRIP_W")) ctx->strip_w = std::atoi(e);
  if (const char* e = std::getenv("PINT_RESID_ACC")) ctx->resid_acc32 = std::string(e) == "f32";
  if (const char* e = std::getenv("PINT_JAC_MT")) ctx->jac_mt = e[0] == '1';
  if (const char* e = std::getenv("PINT_RES")) ctx->res_strip = std::string(e) == "strip";
  if (const char* e = std::getenv("PINT_RES_WAVES")) ctx->res_waves = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("PINT_FORCING")) ctx->forcing = std::atof(e);
  if (const char* e = std::getenv("PINT_TAIL_STAGE")) ctx->tail_stage = std::atoi(e);
  ctx->fuse_prolong = std::getenv("PINT_FUSE_PROLONG") && std::getenv("PINT_FUSE_PROLONG")[0] == '1';
  if (const char* e = std::getenv("PINT_POLL")) ctx->poll_every = std::max(1, std::atoi(e));
  if (cudaStreamCreateWithFlags(&ctx->stream, cudaStreamNonBlocking) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_in, cudaEventDisableTiming) != cudaSuccess ||
      cudaEventCreateWithFlags(&ctx->ev_out, cudaEventDisableTiming) != cudaSuccess) {
    ctx->err = "stream/event creation failed";
    return PINT_CUDA_ERROR;
  }
  ctx->cells[0] = desc->cells[0];
  ctx->cells[1] = desc->cells[1];
  ctx->cells[2] = desc->dim == 3 ? desc->cells[2] : 1;
  ctx->g = make_grid(ctx->D, ctx->cells);
  Phys& ph = ctx->ph;
  ph.rho_f = desc->rho_f;
  ph.rnu = desc->rho_f * desc->nu_f;
  ph.rho_s = desc->rho_s;
  ph.mu = desc->mu_s;
  ph.lam = desc->lambda_s;
  double wq = 1.0, wf = 1.0;
  for (int m = 0; m < 3; ++m) {
    ph.h[m] = m < ctx->D ? desc->extent[m] / desc->cells[m] : 1.0;
    ph.ih[m] = 1.0 / ph.h[m];
    if (m < ctx->D) wq *= 0.5 * ph.h[m];
    if (m >= 1 && m < ctx->D) wf *= 0.5 * ph.h[m];
  }
  ph.wq = wq;
  ph.wf = wf;
  build_tables(ctx);

  const int C = ctx->C;
  const int S = max_slices;
  const size_t vsz = (size_t)C * ctx->g.np;
  int rc;
#define ALLOC(p, cnt)                   \
  if ((rc = dalloc(ctx, &(p), (cnt))) != PINT_OK) return rc;
  ALLOC(ctx->d_node_flags, (size_t)ctx->g.nn);
  ALLOC(ctx->d_cell_flags, ctx->h_cell_flags.size());
  ALLOC(ctx->d_profile, (size_t)ctx->g.nn);
  cudaMemcpy(ctx->d_node_flags, ctx->h_node_flags.data(), ctx->h_node_flags.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(ctx->d_cell_flags, ctx->h_cell_flags.data(), ctx->h_cell_flags.size(), cudaMemcpyHostToDevice);
  cudaMemcpy(ctx->d_profile, ctx->h_profile.data(), sizeof(double) * ctx->h_profile.size(), cudaMemcpyHostToDevice);

  // multigrid hierarchy: coarsen while every cell count is even
  int cl[3] = {ctx->cells[0], ctx->cells[1], ctx->cells[2]};
  for (;;) {
    Level L;
    L.g = make_grid(ctx->D, cl);
    ctx->lv.push_back(L);
    if (ctx->matrix_free) break;  // no hierarchy: level 0's grid only, nothing allocated
    bool even = true;
    for (int m = 0; m < ctx->D; ++m) even = even && (cl[m] % 2 == 0) && cl[m] >= 2;
    if (!even) break;
    for (int m = 0; m < ctx->D; ++m) cl[m] /= 2;
  }
  for (size_t l = 0; l < (ctx->matrix_free ? 0 : ctx->lv.size()); ++l) {
    Level& L = ctx->lv[l];
    const size_t np = L.g.np;
    ALLOC(L.A, (size_t)S * L.g.noff * C * C * np);
    ALLOC(L.Dinv, (size_t)S * C * C * np);
    ALLOC(L.xa, (size_t)S * C * np);
    ALLOC(L.xb, (size_t)S * C * np);
    ALLOC(L.res, (size_t)S * C * np);
    if (l > 0) ALLOC(L.rhs, (size_t)S * C * np);
    if (l > 0) ALLOC(L.sol, (size_t)S * C * np);
    {
      int cl2[3] = {L.g.n[0] - 1, L.g.n[1] - 1, ctx->D == 3 ? L.g.n[2] - 1 : 1};
      L.ncell = cl2[0] * cl2[1] * cl2[2];
      const size_t Lc = (size_t)(1 << ctx->D) * C;
      ALLOC(L.vinv, (size_t)S * Lc * Lc * L.ncell);
      ALLOC(L.ycell, (size_t)S * Lc * L.ncell);
    }
  }
  const Level& Lc = ctx->lv.back();
  // dense buffer sized for the largest level that a max_levels choice could make
  // the coarsest and that still fits kDenseMax dofs
  ctx->dense_cap = 0;
  for (const Level& L : ctx->lv)
    if (ctx->matrix_free) break;
    else
    if (C * L.g.nn <= kDenseMax) ctx->dense_cap = std::max(ctx->dense_cap, C * L.g.nn);
  if (!ctx->matrix_free && ctx->dense_cap == 0 && C * Lc.g.nn <= kDenseMax) ctx->dense_cap = C * Lc.g.nn;
  if (ctx->dense_cap > 0) {
    ALLOC(ctx->d_dense, (size_t)S * ctx->dense_cap * 2 * ctx->dense_cap);
    ALLOC(ctx->d_dense32, (size_t)S * ctx->dense_cap * ((ctx->dense_cap + 3) / 4 * 4));
  }

  ALLOC(ctx->ystate, S * vsz);
  ALLOC(ctx->ynew, S * vsz);
  ALLOC(ctx->r, S * vsz);
  ALLOC(ctx->dx, S * vsz);
  ALLOC(ctx->ytrial, S * vsz);
  ALLOC(ctx->rtrial, S * vsz);
  ALLOC(ctx->b, S * vsz);
  const int m = restart;
  ALLOC(ctx->V, (size_t)(m + 1) * S * vsz);
  if (ctx->matrix_free) ctx->Z = ctx->V;  // no preconditioner: z_j = v_j
  else ALLOC(ctx->Z, (size_t)m * S * vsz);
  ALLOC(ctx->w, S * vsz);
  ALLOC(ctx->u, S * vsz);
  ALLOC(ctx->H, (size_t)S * (m + 1) * m);
  ALLOC(ctx->gv, (size_t)S * (m + 1));
  ALLOC(ctx->cs, (size_t)S * m);
  ALLOC(ctx->sn, (size_t)S * m);
  ALLOC(ctx->ybuf, (size_t)S * (m + 1));
  ALLOC(ctx->gm_res, (size_t)S);
  ALLOC(ctx->gm_tol, (size_t)S);
  ALLOC(ctx->gm_beta, (size_t)S);
  ALLOC(ctx->gm_active, (size_t)S);
  ALLOC(ctx->gm_steps, (size_t)S);
  ALLOC(ctx->gm_its, (size_t)S);
  ALLOC(ctx->cyc_active, (size_t)S);
  ALLOC(ctx->gm_two_pass, (size_t)S);
  ALLOC(ctx->gm_hnorm, (size_t)S);
  ALLOC(ctx->ctr_mdot, (size_t)S);
  ALLOC(ctx->ctr_norm, (size_t)S);
  ctx->nblk = (int)((vsz + kRedChunk - 1) / kRedChunk);
  ALLOC(ctx->partial, (size_t)S * (m + 1) * ctx->nblk);
  ALLOC(ctx->d_norms, (size_t)S);
  ALLOC(ctx->d_degen, (size_t)S);
  ALLOC(ctx->d_active, (size_t)S);
  ALLOC(ctx->d_mask2, (size_t)S);
  ALLOC(ctx->d_lam, (size_t)S);
  ALLOC(ctx->d_st, (size_t)S);
  ALLOC(ctx->d_work, (size_t)1);
  ALLOC(ctx->d_work_bytes, (size_t)1);
  ALLOC(ctx->cpart, (size_t)S * kTailCluster * kMaxBasis);
#undef ALLOC
  // optional fp32 copy of the level-0 operator for the V-cycle residuals (half
  // the bytes of the two level-0 SpMVs of every cycle); skipped when it does
  // not fit next to the rest of the workspace (or with PINT_A32=0)
  // The coarse levels that run as standalone kernels (above the fused tail)
  // get an fp32 copy too (made after their Galerkin product; PINT_A32C=0 keeps
  // them fp64): their V-cycle residual SpMVs were 8 % of the c3 step in fp64.
  if (!ctx->matrix_free && !(std::getenv("PINT_A32") && std::getenv("PINT_A32")[0] == '0')) {
    const bool coarse = !(std::getenv("PINT_A32C") && std::getenv("PINT_A32C")[0] == '0');
    for (size_t l = 0; l < (coarse ? ctx->lv.size() : 1); ++l) {
      Level& L = ctx->lv[l];
      if (l > 0 && (size_t)L.g.nn * C <= (size_t)ctx->tail_rows) break;  // the tail reads fp64 there
      const size_t cnt = (size_t)S * L.g.noff * C * C * L.g.np;
      size_t free_b = 0, total_b = 0;
      if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || cnt * sizeof(float) + (size_t(2) << 30) >= free_b)
        break;
      if (dalloc(ctx, &L.A32, cnt) != PINT_OK) {
        L.A32 = nullptr;
        ctx->err.clear();
        cudaGetLastError();
        break;
      }
    }
  }
  // Vanka sweeps in block-stencil form on every level (standalone kernels and
  // the fused tail); without room for it the cell-inverse sweeps stay
  // (PINT_VANKA=fused|split force them)
  if (!ctx->matrix_free && ctx->vanka_stencil) {
    for (size_t l = 0; l < ctx->lv.size(); ++l) {
      Level& L = ctx->lv[l];
      const size_t cnt = (size_t)S * L.g.noff * C * C * L.g.np;
      size_t free_b = 0, total_b = 0;
      if (cudaMemGetInfo(&free_b, &total_b) != cudaSuccess || cnt * sizeof(float) + (size_t(2) << 30) >= free_b)
        break;
      if (dalloc(ctx, &L.vst, cnt) != PINT_OK) {
        L.vst = nullptr;
        ctx->err.clear();
        cudaGetLastError();
        break;
      }
    }
  }
  if (ctx->lv.empty() || !ctx->lv[0].vst) ctx->vanka_stencil = false;
  if (ctx->vanka_stencil) ctx->vanka_split = false;
  // device-driven control flow: per-slice loop state
  {
    LoopDev& d = ctx->ld;
    int rc2;
#define LALLOC(p, cnt) \
  if ((rc2 = dalloc(ctx, &(p), (cnt))) != PINT_OK) return rc2;
    LALLOC(d.ls, (size_t)1);
    for (int** q : {&d.act, &d.status, &d.nit, &d.kit, &d.running, &d.its, &d.ls_mask, &d.accept, &d.ok, &d.built,
                    &d.base, &d.first, &d.need, &d.built_now, &d.gits})
      LALLOC(*q, (size_t)S);
    for (double** q : {&d.ft, &d.rnorm, &d.target, &d.tnorm, &d.lam, &d.gres}) LALLOC(*q, (size_t)S);
    LALLOC(ctx->gm_cap, (size_t)1);
    LALLOC(ctx->d_body_nodes, (size_t)kMaxBodies);
    LALLOC(ctx->d_launch_ctr, (size_t)1);
#undef LALLOC
    d.gm_tol = ctx->gm_tol;
    d.gm_beta = ctx->gm_beta;
    d.gv = ctx->gv;
    d.norms = ctx->d_norms;
    d.gm_active = ctx->gm_active;
    d.gm_steps = ctx->gm_steps;
    d.gm_its = ctx->gm_its;
    d.cyc_active = ctx->cyc_active;
    d.gm_two_pass = ctx->gm_two_pass;
    d.gm_cap = ctx->gm_cap;
    d.st = ctx->d_st;
    d.launch_ctr = ctx->d_launch_ctr;
    d.body_nodes = ctx->d_body_nodes;
    for (int i = 0; i < kCapDepth; ++i)
      if (cudaStreamCreateWithFlags(&ctx->cap_st[i], cudaStreamNonBlocking) != cudaSuccess) {
        ctx->err = "capture stream creation failed";
        return PINT_CUDA_ERROR;
      }
  }
  ctx->device_loop = !(std::getenv("PINT_DEVICE_LOOP") && std::getenv("PINT_DEVICE_LOOP")[0] == '0');
  if (const char* e = std::getenv("PINT_GATE")) ctx->gate = std::max(1, std::atoi(e));
  if (const char* e = std::getenv("PINT_GATE0")) ctx->gate0 = std::max(0, std::atoi(e));
  if (cudaMallocHost(&ctx->h_dbl, sizeof(double) * S) != cudaSuccess ||
      cudaMallocHost(&ctx->h_int, sizeof(int) * S) != cudaSuccess ||
      cudaMallocHost(&ctx->h_cap, sizeof(int)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_ls, sizeof(LoopScalars)) != cudaSuccess ||
      cudaMallocHost(&ctx->h_out_i, sizeof(int) * 4 * S) != cudaSuccess ||
      cudaMallocHost(&ctx->h_out_d, sizeof(double) * S) != cudaSuccess) {
    ctx->err = "cudaMallocHost failed";
    return PINT_CUDA_ERROR;
  }
  cudaError_t e = cudaDeviceSynchronize();
  if (e != cudaSuccess) {
    ctx->err = std::string("create: ") + cudaGetErrorString(e);
    return PINT_CUDA_ERROR;
  }
  return PINT_OK;
}

int pint_destroy(pint_ctx* ctx) {
  if (!ctx) return PINT_OK;
  cudaDeviceSynchronize();
  for (void* p : ctx->allocs) cudaFree(p);
  for (cudaEvent_t e : ctx->ev_pool) cudaEventDestroy(e);
  for (auto& kv : ctx->graphs) cudaGraphExecDestroy(kv.second.first);
  for (auto& kv : ctx->loop_graphs) cudaGraphExecDestroy(kv.second.first);
  for (void* p : {(void*)ctx->d_sts, (void*)ctx->d_t1tab, (void*)ctx->d_nsteps, (void*)ctx->d_lsv,
                  (void*)ctx->sw_part, (void*)ctx->sw_theta, (void*)ctx->sw_corr, (void*)ctx->sw_ft,
                  (void*)ctx->sw_status, (void*)ctx->sw_nit, (void*)ctx->sw_kit})
    if (p) cudaFree(p);
  for (void* p : {(void*)ctx->h_sts, (void*)ctx->h_t1tab, (void*)ctx->h_nsteps, (void*)ctx->h_lsv,
                  (void*)ctx->h_sw, (void*)ctx->h_cap, (void*)ctx->h_ls, (void*)ctx->h_out_i, (void*)ctx->h_out_d})
    if (p) cudaFreeHost(p);
  for (cudaStream_t cs : ctx->cap_st)
    if (cs) cudaStreamDestroy(cs);
  if (ctx->stream) cudaStreamDestroy(ctx->stream);
  if (ctx->ev_in) cudaEventDestroy(ctx->ev_in);
  if (ctx->ev_out) cudaEventDestroy(ctx->ev_out);
  if (ctx->h_dbl) cudaFreeHost(ctx->h_dbl);
  if (ctx->h_int) cudaFreeHost(ctx->h_int);
  delete ctx;
  return PINT_OK;
}

const char* pint_last_error(const pint_ctx* ctx) { return ctx ? ctx->err.c_str() : "null context"; }

int pint_sizes(const pint_ctx* ctx, int32_t* nn, int32_t* np, int32_t* C, int32_t* levels) {
  if (!ctx) return PINT_INVALID_ARG;
  if (nn) *nn = ctx->g.nn;
  if (np) *np = ctx->g.np;
  if (C) *C = ctx->C;
  if (levels) *levels = (int32_t)ctx->lv.size();
  return PINT_OK;
}

int pint_level0_fp32(const pint_ctx* ctx, int32_t* enabled) {
  if (!ctx || !enabled) return PINT_INVALID_ARG;
  *enabled = ctx->lv.empty() || !ctx->lv[0].A32 ? 0 : 1;
  return PINT_OK;
}

int pint_flags(const pint_ctx* ctx, uint8_t* node_flags, uint8_t* cell_flags) {
  if (!ctx) return PINT_INVALID_ARG;
  if (node_flags) std::memcpy(node_flags, ctx->h_node_flags.data(), ctx->h_node_flags.size());
  if (cell_flags) std::memcpy(cell_flags, ctx->h_cell_flags.data(), ctx->h_cell_flags.size());
  return PINT_OK;
}

int pint_profile(pint_ctx* ctx, int32_t enable) {
  if (!ctx) return PINT_INVALID_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  cudaDeviceSynchronize();
  ctx->prof = enable == 2;  // 1: count launches only (graphs stay on); 2: + CUDA events around the kernel
  ctx->launches = 0;
  ctx->ev_pairs.clear();
  ctx->ev_used = 0;
  cudaMemset(ctx->d_work, 0, sizeof(unsigned long long));
  cudaMemset(ctx->d_work_bytes, 0, sizeof(unsigned long long));
  if (ctx->d_launch_ctr) cudaMemset(ctx->d_launch_ctr, 0, sizeof(unsigned long long));
  ctx->fused_used = false;
  ctx->tail_slice_launches = 0;
  return PINT_OK;
}

const char* pint_profile_kernel(const pint_ctx* ctx) {
  if (!ctx) return "";
  if (ctx->fused_used) return ctx->D == 2 ? "k_arnoldi_fused<2> (whole Arnoldi step: V-cycle + SpMV + CGS2 + Givens)"
                                         : "k_arnoldi_fused<3> (whole Arnoldi step: V-cycle + SpMV + CGS2 + Givens)";
  if (ctx->tail_first == 0)
    return ctx->D == 2 ? "k_vcycle_tail_cl<2> (whole V-cycle: mesh fits the cluster tail)"
                       : "k_vcycle_tail_cl<3> (whole V-cycle: mesh fits the cluster tail)";
  if (ctx->kopt.smoother == 1 && ctx->vanka_stencil)
    return ctx->D == 2 ? "k_vanka_stencil_apply<2> (level-0 Vanka sweep as one fp32 block-stencil product)"
                       : "k_vanka_stencil_apply<3> (level-0 Vanka sweep as one fp32 block-stencil product)";
  if (ctx->kopt.smoother == 1 && ctx->vanka_split)
    return ctx->D == 2 ? "k_vanka_cell<2,16> (level-0 cell-patch Vanka solves)"
                       : "k_vanka_cell<3,8> (level-0 cell-patch Vanka solves)";
  if (ctx->kopt.smoother == 1) return ctx->D == 2 ? "k_vanka_apply<2> (level-0 Vanka sweep: cell solves + gather)"
                                                  : "k_vanka_apply<3> (level-0 Vanka sweep: cell solves + gather)";
  return ctx->D == 2 ? "k_smooth<2,false> (level-0 node-block Jacobi sweep)" : "k_smooth<3,false>";
}

int pint_profile_read(pint_ctx* ctx, int64_t* launches, int64_t* kernel_launches, int64_t* slice_launches,
                      double* kernel_ms, int64_t* bytes_per_slice_launch) {
  if (!ctx) return PINT_INVALID_ARG;
  std::lock_guard<std::mutex> lock(ctx->mu);
  PINT_CHECK(cudaDeviceSynchronize());
  double ms = 0.0;
  for (auto& pr : ctx->ev_pairs) {
    float t = 0.f;
    cudaEventElapsedTime(&t, pr.first, pr.second);
    ms += t;
  }
  unsigned long long work = 0;
  PINT_CHECK(cudaMemcpy(&work, ctx->d_work, sizeof(work), cudaMemcpyDeviceToHost));
  unsigned long long dev_launches = 0;  // kernels inside the conditional bodies of the loop graphs
  PINT_CHECK(cudaMemcpy(&dev_launches, ctx->d_launch_ctr, sizeof(dev_launches), cudaMemcpyDeviceToHost));
  if (launches) *launches = ctx->launches + (int64_t)dev_launches;
  if (kernel_launches) *kernel_launches = (int64_t)ctx->ev_pairs.size();
  const bool tail_kernel = !ctx->fused_used && ctx->tail_first == 0;
  if (slice_launches) *slice_launches = tail_kernel ? ctx->tail_slice_launches : (int64_t)work;
  if (kernel_ms) *kernel_ms = ms;
  if (bytes_per_slice_launch && ctx->fused_used) {
    unsigned long long wb = 0;
    PINT_CHECK(cudaMemcpy(&wb, ctx->d_work_bytes, sizeof(wb), cudaMemcpyDeviceToHost));
    *bytes_per_slice_launch = work ? (int64_t)(wb / work) : 0;  // k_arnoldi_fused, averaged over j
  } else if (bytes_per_slice_launch && tail_kernel) {
    *bytes_per_slice_launch =
        (int64_t)(ctx->D == 2 ? Impl<2>::vcycle_bytes(ctx, 0) : Impl<3>::vcycle_bytes(ctx, 0));
  } else if (bytes_per_slice_launch) {
    const Grid& g = ctx->lv[0].g;
    const int64_t C = ctx->C;
    if (ctx->kopt.smoother == 1 && ctx->vanka_stencil) {
      // k_vanka_stencil_apply: fp32 stencil (noff C^2 per node) + residual in + x out (C per node each);
      // the x_in read of the non-first sweeps is not counted (lower bound)
      *bytes_per_slice_launch = (int64_t)g.nn * (4 * (int64_t)g.noff * C * C + 16 * C);
    } else if (ctx->kopt.smoother == 1 && ctx->vanka_split) {
      // k_vanka_cell: cell inverses (L^2) + cell corrections (L) per cell, residual C per node
      const int64_t Lc = (int64_t)(1 << ctx->D) * C;
      *bytes_per_slice_launch = (int64_t)ctx->lv[0].ncell * (4 * Lc * Lc + 8 * Lc) + (int64_t)g.nn * 8 * C;
    } else if (ctx->kopt.smoother == 1) {
      // k_vanka_apply: fp32 cell inverses (L^2 per cell) + residual in + x out (C per node each);
      // the x_in read of the non-first sweeps is not counted (lower bound)
      const int64_t Lc = (int64_t)(1 << ctx->D) * C;
      *bytes_per_slice_launch = (int64_t)ctx->lv[0].ncell * 4 * Lc * Lc + (int64_t)g.nn * 16 * C;
    } else {
      // k_smooth: A (noff C^2) + Dinv (C^2) + b + x_in + x_out (3 C), fp64, per node
      *bytes_per_slice_launch = (int64_t)g.nn * 8 * ((int64_t)g.noff * C * C + C * C + 3 * C);
    }
  }
  return PINT_OK;
}

#define DISPATCH(call) (ctx->D == 2 ? Impl<2>::call : Impl<3>::call)

int pint_propagate(pint_ctx* ctx, int32_t S, const double* y_in, double* y_out, const double* t0,
                   const double* t_end, const int32_t* nsteps, double k, double theta0,
                   const pint_newton_opts* newton, const pint_krylov_opts* krylov, int32_t* newton_iters,
                   int32_t* krylov_iters, int32_t* status, double* fail_t, void* stream) {
  int rc = check_S(ctx, S);
  if (rc) return rc;
  if (!y_in || !y_out || !t0 || !t_end || !nsteps || !newton || !krylov || k <= 0.0) {
    ctx->err = "invalid argument to pint_propagate";
    return PINT_INVALID_ARG;
  }
  if (krylov->restart != ctx->restart) {
    ctx->err = "krylov restart " + std::to_string(krylov->restart) + " differs from the context's restart length " +
               std::to_string(ctx->restart);
    return PINT_INVALID_ARG;
  }
  if (ctx->matrix_free) return mf_reject(ctx, "pint_propagate");
  std::lock_guard<std::mutex> lock(ctx->mu);
  StreamGuard guard(ctx, stream);
  cudaStream_t st = ctx->stream;
  if (use_device_loop(ctx))
    return propagate_dev(ctx, S, y_in, y_out, t0, t_end, nsteps, k, theta0, newton, krylov, newton_iters,
                         krylov_iters, status, fail_t, st);
  return DISPATCH(propagate(ctx, S, y_in, y_out, t0, t_end, nsteps, k, theta0, newton, krylov, newton_iters,
                            krylov_iters, status, fail_t, st));
}

int pint_residual(pint_ctx* ctx, int32_t S, const double* y, const double* y_old, const double* k,
                  const double* theta, const double* t1, double* r, double* norms, void* stream) {
  int rc = check_S(ctx, S);
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(ctx->mu);
  StreamGuard guard(ctx, stream);
  cudaStream_t st = ctx->stream;
  if ((rc = upload_steps(ctx, S, k, theta, t1, st))) return rc;
  std::vector<double> tmp(S);
  rc = DISPATCH(residual(ctx, S, y, y_old, r, nullptr, tmp.data(), st));
  if (rc == PINT_OK && norms) std::memcpy(norms, tmp.data(), sizeof(double) * S);
  return rc;
}

int pint_jvp(pint_ctx* ctx, int32_t S, const double* y, const double* y_old, const double* w, const double* k,
             const double* theta, const double* t1, double* Jw, void* stream) {
  int rc = check_S(ctx, S);
  if (rc) return rc;
  std::lock_guard<std::mutex> lock(ctx->mu);
  StreamGuard guard(ctx, stream);
  cudaStream_t st = ctx->stream;
  if ((rc = upload_steps(ctx, S, k, theta, t1, st))) return rc;
  return DISPATCH(jvp(ctx, S, y, y_old, w, Jw, st));
}

int pint_assemble(pint_ctx* ctx, int32_t S, const double* y, const double* y_old, const double* k,
                  const double* theta, const double* t1, void* stream) {
  int rc = check_S(ctx, S);
  if (rc) return rc;
  if (ctx->matrix_free) return mf_reject(ctx, "pint_assemble");
  std::lock_guard<std::mutex> lock(ctx->mu);
  StreamGuard guard(ctx, stream);
  cudaStream_t st = ctx->stream;
  if ((rc = upload_steps(ctx, S, k, theta, t1, st))) return rc;
  return DISPATCH(assemble(ctx, S, y, y_old, nullptr, st));
}

int pint_jacobian_blocks(pint_ctx* ctx, int32_t S, double* out, void* stream) {
  int rc = check_S(ctx, S);
  if (rc) return rc;
  if (ctx->matrix_free) return mf_reject(ctx, "pint_jacobian_blocks");
  std::lock_guard<std::mutex> lock(ctx->mu);
  const size_t ms = (size_t)ctx->g.noff * ctx->C * ctx->C * ctx->g.np;
  StreamGuard guard(ctx, stream);
  PINT_CHECK(cudaMemcpyAsync(out, ctx->lv[0].A, sizeof(double) * ms * S, cudaMemcpyDeviceToDevice, ctx->stream));
  return PINT_OK;
}

int pint_spmv(pint_ctx* ctx, int32_t S, const double* x, double* y, void* stream) {
  int rc = check_S(ctx, S);
  if (rc) return rc;
  if (ctx->matrix_free) return mf_reject(ctx, "pint_spmv");
  std::lock_guard<std::mutex> lock(ctx->mu);
  StreamGuard guard(ctx, stream);
  DISPATCH(spmv(ctx, 0, S, x, y, nullptr, ctx->stream));
  PINT_LAUNCHED();
  return PINT_OK;
}

int pint_precond_setup(pint_ctx* ctx, int32_t S, const pint_krylov_opts* krylov, void* stream) {
  int rc = check_S(ctx, S);
  if (rc) return rc;
  if (ctx->matrix_free) return mf_reject(ctx, "pint_precond_setup");
  std::lock_guard<std::mutex> lock(ctx->mu);
  StreamGuard guard(ctx, stream);
  return DISPATCH(precond_setup(ctx, S, krylov, nullptr, ctx->stream));
}

int pint_precond_apply(pint_ctx* ctx, int32_t S, const double* b, double* x, void* stream) {
  int rc = check_S(ctx, S);
  if (rc) return rc;
  if (ctx->matrix_free) return mf_reject(ctx, "pint_precond_apply");
  std::lock_guard<std::mutex> lock(ctx->mu);
  if (ctx->prec_levels == 0) {
    ctx->err = "pint_precond_apply before pint_precond_setup";
    return PINT_INVALID_ARG;
  }
  StreamGuard guard(ctx, stream);
  DISPATCH(vcycle(ctx, 0, S, b, x, nullptr, ctx->stream));
  PINT_LAUNCHED();
  return PINT_OK;
}

int pint_linear_solve(pint_ctx* ctx, int32_t S, const double* b, double* x, const pint_krylov_opts* krylov,
                      int32_t* its, double* resid, void* stream) {
  int rc = check_S(ctx, S);
  if (rc) return rc;
  if (krylov->restart != ctx->restart) {
    ctx->err = "krylov restart " + std::to_string(krylov->restart) + " differs from the context's restart length " +
               std::to_string(ctx->restart);
    return PINT_INVALID_ARG;
  }
  if (ctx->matrix_free) return mf_reject(ctx, "pint_linear_solve");
  std::lock_guard<std::mutex> lock(ctx->mu);
  StreamGuard guard(ctx, stream);
  return DISPATCH(gmres(ctx, S, b, x, nullptr, krylov, nullptr, nullptr, its, resid, ctx->stream));
}

int pint_linear_solve_mf(pint_ctx* ctx, int32_t S, const double* y, const double* y_old, const double* k,
                         const double* theta, const double* t1, const double* b, double* x,
                         const pint_krylov_opts* krylov, int32_t* its, double* resid, void* stream) {
  int rc = check_S(ctx, S);
  if (rc) return rc;
  if (!y || !y_old || !k || !theta || !t1 || !b || !x || !krylov) {
    ctx->err = "invalid argument to pint_linear_solve_mf";
    return PINT_INVALID_ARG;
  }
  if (krylov->restart != ctx->restart) {
    ctx->err = "krylov restart " + std::to_string(krylov->restart) + " differs from the context's restart length " +
               std::to_string(ctx->restart);
    return PINT_INVALID_ARG;
  }
  std::lock_guard<std::mutex> lock(ctx->mu);
  StreamGuard guard(ctx, stream);
  cudaStream_t st = ctx->stream;
  if ((rc = upload_steps(ctx, S, k, theta, t1, st))) return rc;
  // an assembled context solves matrix-free too, with its preconditioner off
  const bool was_mf = ctx->matrix_free;
  ctx->matrix_free = true;
  ctx->mf_y = y;
  ctx->mf_yo = y_old;
  double* Zsave = ctx->Z;
  ctx->Z = ctx->V;
  rc = DISPATCH(gmres(ctx, S, b, x, nullptr, krylov, nullptr, nullptr, its, resid, st));
  ctx->Z = Zsave;
  ctx->matrix_free = was_mf;
  ctx->mf_y = ctx->mf_yo = nullptr;
  return rc;
}

int pint_parareal_precorrect(int32_t S, int32_t C, int32_t nn, int32_t np, const double* f_old,
                             const double* c_old, double* delta, void* stream) {
  if (S < 1 || C < 1 || nn < 1 || np < nn) return PINT_INVALID_ARG;
  const size_t total = (size_t)S * C * np;
  size_t blocks = std::min<size_t>((total + 255) / 256, 4096);
  k_precorrect<<<(unsigned)blocks, 256, 0, (cudaStream_t)stream>>>(f_old, c_old, delta, total);
  return cudaGetLastError() == cudaSuccess ? PINT_OK : PINT_CUDA_ERROR;
}

int pint_parareal_correct_one(int32_t C, int32_t nn, int32_t np, const double* c_new, const double* f_old,
                              const double* c_old, const double* x_prev, double* x_new, int32_t variant,
                              double clamp_lo, double clamp_hi, double* theta_out, double* corr_out,
                              void* stream) {
  if (C < 1 || nn < 1 || np < nn || variant < 0 || variant > 2 || clamp_lo > clamp_hi) return PINT_INVALID_ARG;
  cudaStream_t st = (cudaStream_t)stream;
  const int nblk = (nn + kRedChunk - 1) / kRedChunk;
  // scratch of the largest call so far (process-wide, serialised by its mutex)
  static std::mutex mu;
  static double* scratch = nullptr;
  static size_t scratch_cnt = 0;
  std::lock_guard<std::mutex> lock(mu);
  const size_t cnt = (size_t)C * 3 * nblk + (size_t)C * 2 * nblk + 2;
  if (cnt > scratch_cnt) {
    if (scratch) cudaFree(scratch);
    scratch = nullptr;
    if (cudaMalloc((void**)&scratch, sizeof(double) * cnt) != cudaSuccess) {
      scratch_cnt = 0;
      return PINT_CUDA_ERROR;
    }
    scratch_cnt = cnt;
  }
  double* part3 = scratch;
  double* part2 = scratch + (size_t)C * 3 * nblk;
  double* d_theta = part2 + (size_t)C * 2 * nblk;
  double* d_corr = d_theta + 1;
  k_block_dots<<<dim3(nblk, C), kRedThreads, 0, st>>>(f_old, c_new, nn, np, part3, nblk);
  k_theta<<<1, 32, 0, st>>>(part3, nblk, C, variant, clamp_lo, clamp_hi, d_theta);
  k_update_norms<<<dim3(nblk, C), kRedThreads, 0, st>>>(c_new, f_old, c_old, x_prev, x_new, d_theta, nn, np, part2,
                                                        nblk);
  k_corr<<<1, 32, 0, st>>>(part2, nblk, C, d_corr);
  double hres[2];
  cudaMemcpyAsync(hres, d_theta, sizeof(double) * 2, cudaMemcpyDeviceToHost, st);
  if (cudaStreamSynchronize(st) != cudaSuccess) return PINT_CUDA_ERROR;
  if (theta_out) *theta_out = hres[0];
  if (corr_out) *corr_out = hres[1];
  return cudaGetLastError() == cudaSuccess ? PINT_OK : PINT_CUDA_ERROR;
}

int pint_coarse_sweep(pint_ctx* ctx, int32_t L, double* x, const double* x_prev, double* c_new, const double* c_old,
                      const double* f_old, const double* t_grid, const int32_t* nsteps, double k, double theta0,
                      const pint_newton_opts* newton, const pint_krylov_opts* krylov, int32_t variant,
                      double clamp_lo, double clamp_hi, double* theta_out, double* corr_out, int32_t* newton_iters,
                      int32_t* krylov_iters, int32_t* status, double* fail_t, void* stream) {
  if (!ctx) return PINT_INVALID_ARG;
  if (L < 1 || !x || !c_new || !t_grid || !nsteps || !newton || !krylov || k <= 0.0 || variant < 0 || variant > 2 ||
      clamp_lo > clamp_hi || (f_old && (!c_old || !x_prev))) {
    ctx->err = "invalid argument to pint_coarse_sweep";
    return PINT_INVALID_ARG;
  }
  if (krylov->restart != ctx->restart) {
    ctx->err = "krylov restart " + std::to_string(krylov->restart) + " differs from the context's restart length " +
               std::to_string(ctx->restart);
    return PINT_INVALID_ARG;
  }
  for (int l = 0; l < L; ++l)
    if (nsteps[l] < 0 || !(t_grid[l + 1] >= t_grid[l])) {
      ctx->err = "pint_coarse_sweep: time grid must be non-decreasing with non-negative step counts";
      return PINT_INVALID_ARG;
    }
  if (ctx->matrix_free) return mf_reject(ctx, "pint_coarse_sweep");
  std::lock_guard<std::mutex> lock(ctx->mu);
  StreamGuard guard(ctx, stream);
  return coarse_sweep(ctx, L, x, x_prev, c_new, c_old, f_old, t_grid, nsteps, k, theta0, newton, krylov, variant,
                      clamp_lo, clamp_hi, theta_out, corr_out, newton_iters, krylov_iters, status, fail_t,
                      ctx->stream);
}

int pint_boundary_error(pint_ctx* ctx, int32_t S, const double* x, const double* ref, double* err,
                        int32_t* absolute, void* stream) {
  if (!ctx) return PINT_INVALID_ARG;
  if (S < 1 || !x || !ref || !err) {
    ctx->err = "invalid argument to pint_boundary_error";
    return PINT_INVALID_ARG;
  }
  std::lock_guard<std::mutex> lock(ctx->mu);
  StreamGuard guard(ctx, stream);
  cudaStream_t st = ctx->stream;
  PINT_TRY(ensure_sweep(ctx, (size_t)S));
  const size_t n = (size_t)ctx->C * ctx->g.np;
  const int nblk = ctx->nblk;
  pint_launch(ctx, st, k_err_partial, dim3(nblk, S), kRedThreads, 0, x, ref, n, ctx->sw_part, nblk);
  pint_launch(ctx, st, k_err_final, (S + 127) / 128, 128, 0, (const double*)ctx->sw_part, nblk, S, ctx->sw_theta,
              ctx->sw_status);
  PINT_LAUNCHED();
  PINT_CHECK(cudaMemcpyAsync(ctx->h_sw, ctx->sw_theta, sizeof(double) * S, cudaMemcpyDeviceToHost, st));
  int* hi = reinterpret_cast<int*>(ctx->h_sw + 3 * ctx->sw_cap);
  PINT_CHECK(cudaMemcpyAsync(hi, ctx->sw_status, sizeof(int) * S, cudaMemcpyDeviceToHost, st));
  PINT_CHECK(cudaStreamSynchronize(st));
  for (int s = 0; s < S; ++s) {
    err[s] = ctx->h_sw[s];
    if (absolute) absolute[s] = hi[s];
  }
  return PINT_OK;
}

}  // extern "C"
