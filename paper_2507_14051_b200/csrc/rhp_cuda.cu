// rhp_cuda.cu — device context and the C ABI of include/rhpdhg_cuda.h.
//
// One rhp_ctx = one solve's device state on one GPU. Host code here only
// allocates, uploads, builds the CUDA graph and launches; all arithmetic of
// the solve runs in the kernels of pdhg_kernels.cuh.
#include <cuda_profiler_api.h>
#include <cuda_runtime.h>

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <limits>
#include <stdexcept>
#include <string>
#include <thread>
#include <tuple>
#include <vector>

#ifdef RHP_WITH_NCCL
#include <dlfcn.h>
#include <nccl.h>
#endif

#include "comm.cuh"
#include "ingest.cuh"
#include "layout.cuh"
#include "op_kernels.cuh"
#include "pdhg_kernels.cuh"
#include "peer.cuh"
#include "resident.cuh"
#include "scaling_kernels.cuh"
#include "segments.cuh"
#include "rhpdhg_cuda.h"

using namespace rhp;

namespace {

thread_local std::string g_err;

using CudaError = rhp::DeviceFailure;

void check(cudaError_t e, const char* what) {
  if (e != cudaSuccess)
    throw CudaError(std::string(what) + ": " + cudaGetErrorName(e) + " (" + cudaGetErrorString(e) + ")");
}
#define CK(call) check((call), #call)

#ifdef RHP_WITH_NCCL
// NCCL is resolved at run time (dlopen of libnccl.so.2) rather than linked:
// a single-GPU user never loads it, and in a process where PyTorch already
// loaded its own NCCL the same library is reused — linking the system copy
// would shadow torch's newer one and break `import torch` afterwards.
struct NcclApi {
  decltype(&ncclGetUniqueId) GetUniqueId = nullptr;
  decltype(&ncclCommInitRank) CommInitRank = nullptr;
  decltype(&ncclCommDestroy) CommDestroy = nullptr;
  decltype(&ncclAllReduce) AllReduce = nullptr;
  decltype(&ncclAllGather) AllGather = nullptr;
  decltype(&ncclReduceScatter) ReduceScatter = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api = [] {
    NcclApi a;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) return a;
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(dlsym(h, "ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(dlsym(h, "ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(dlsym(h, "ncclCommDestroy"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(dlsym(h, "ncclAllReduce"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(dlsym(h, "ncclAllGather"));
    a.ReduceScatter = reinterpret_cast<decltype(a.ReduceScatter)>(dlsym(h, "ncclReduceScatter"));
    return a;
  }();
  if (!api.GetUniqueId || !api.CommInitRank || !api.CommDestroy || !api.AllReduce || !api.AllGather ||
      !api.ReduceScatter)
    throw rhp::DeviceFailure("NCCL (libnccl.so.2) not found: the row-partitioned path needs it");
  return api;
}

// The production transport of comm.cuh: one NCCL communicator per rank.
class NcclComm final : public rhp::Comm {
 public:
  NcclComm(const void* id128, int world, int rank) {
    ncclUniqueId id;
    std::memcpy(&id, id128, sizeof(id));
    if (nccl().CommInitRank(&comm_, world, id, rank) != ncclSuccess)
      throw CudaError("ncclCommInitRank failed");
  }
  ~NcclComm() override {
    if (comm_) nccl().CommDestroy(comm_);
  }
  void allreduce(double* buf, size_t count, bool max, cudaStream_t s) override {
    if (nccl().AllReduce(buf, buf, count, ncclDouble, max ? ncclMax : ncclSum, comm_, s) != ncclSuccess)
      throw CudaError("ncclAllReduce failed");
  }
  void allreduce_max_i64(int64_t* buf, size_t count, cudaStream_t s) override {
    if (nccl().AllReduce(buf, buf, count, ncclInt64, ncclMax, comm_, s) != ncclSuccess)
      throw CudaError("ncclAllReduce(int64 max) failed");
  }
  void allgather(const void* send, void* recv, size_t bytes, cudaStream_t s) override {
    if (nccl().AllGather(send, recv, bytes, ncclChar, comm_, s) != ncclSuccess)
      throw CudaError("ncclAllGather failed");
  }
  void reduce_scatter(const double* send, double* recv, size_t chunk, cudaStream_t s) override {
    if (nccl().ReduceScatter(send, recv, chunk, ncclDouble, ncclSum, comm_, s) != ncclSuccess)
      throw CudaError("ncclReduceScatter failed");
  }
  bool is_nccl() const override { return true; }

 private:
  ncclComm_t comm_ = nullptr;
};
#endif

template <class F>
int guarded(F&& f) {
  try {
    f();
    return RHPDHG_OK;
  } catch (const CudaError& e) {
    g_err = e.what();
    return RHPDHG_E_DEVICE;
  } catch (const std::out_of_range& e) {
    g_err = e.what();
    return RHPDHG_E_USAGE;
  } catch (const std::invalid_argument& e) {
    g_err = e.what();
    return RHPDHG_E_USAGE;
  } catch (const std::domain_error& e) {
    g_err = e.what();
    return RHPDHG_E_INVALID_PROBLEM;
  } catch (const std::exception& e) {
    g_err = e.what();
    return RHPDHG_E_INTERNAL;
  }
}

// Every device array gets 64 B of zeroed tail padding (ingest.cuh).
template <class T>
T* dev_alloc(size_t count) {
  return dev_alloc_zero<T>(count);
}

template <class T>
void upload(T* dst, const T* src, size_t count, cudaStream_t s) {
  if (count) CK(cudaMemcpyAsync(dst, src, count * sizeof(T), cudaMemcpyHostToDevice, s));
}

struct DevOp : DeviceCsr {
  Sched sched{};  // with device pointers
  int64_t *warp_row = nullptr, *warp_nz = nullptr, *slot_row = nullptr;
  int32_t *head_slot = nullptr, *tail_slot = nullptr, *slot_first = nullptr, *slot_count = nullptr;
  double *slot_part = nullptr, *long_red = nullptr;
  unsigned int* slot_ticket = nullptr;
  bool l1g = false;  // L1-allocating gathers (choose_gather_policy)
  // column segments (segments.cuh, build_segments): when non-empty the SpMV
  // walks segs[0..S-1] in order, the last one with the real epilogue, and
  // every schedule-dependent use goes through fin() (the last segment)
  std::vector<DevOp> segs;
  double* segbuf = nullptr;  // [rows] running row sums of the segments
  // long-row engine (spmv_cta_rows): CTA b owns rows [cta_row[b], cta_row[b+1])
  int32_t* cta_row = nullptr;
  int cta_grid = 0;  // its own grid (resident CTAs of spmv_cta_rows x SMs, at most one per row)
  // column segments: the row band [seg_rb, seg_re) split by columns; an
  // intermediate segment stores its band-local row sums at seg_out
  int64_t seg_rb = 0, seg_re = 0;
  double* seg_out = nullptr;
  // sliced copy of a uniform thread-per-row operator (Sched::sell_*, build_sliced)
  int32_t* sell_ci = nullptr;
  bool row_band = false;  // a thread-per-row row band runs ahead of the final pass (carve_row_band)
  double* sell_v = nullptr;
  Csr csr() const { return Csr{rp, ci, v, rows}; }
};

}  // namespace

struct rhp_ctx {
  rhp_options opt{};
  int sm_count = 0;
  cudaStream_t stream = nullptr;
  HostLayout L;
  int64_t m = 0, n = 0;
  DevOp A, At;
  // vectors in device (permuted) order
  double *c = nullptr, *vl = nullptr, *vu = nullptr, *cl = nullptr, *cu = nullptr;  // scaled
  double *co = nullptr, *vlo = nullptr, *vuo = nullptr, *clo = nullptr, *cuo = nullptr;
  double *rs = nullptr, *cs = nullptr;
  double *x = nullptr, *y = nullptr, *ax = nullptr, *aty = nullptr;
  double *x0 = nullptr, *y0 = nullptr, *ax0 = nullptr, *aty0 = nullptr;
  double *xp = nullptr, *yp = nullptr;
  double *xout = nullptr, *yout = nullptr, *rcout = nullptr;
  double *pv = nullptr, *pw = nullptr, *pav = nullptr;
  double *part1 = nullptr, *part3 = nullptr, *partA = nullptr, *partAt = nullptr;
  double* hist = nullptr;
  Ctl* ctl = nullptr;
  Ctl* ctl_host = nullptr;  // pinned mirror
  int grid_a = 1, grid_at = 1, grid_vec = 1, grid_max = 1;
  // Row-partitioned: the n-side walkers (block-start primal step, K2c, KKT
  // column sums, power-iteration dots) use this rank-INDEPENDENT map — one
  // column per thread, grid vec_grid(n) — instead of the local A_p^T
  // schedule, whose chunks differ per rank: every rank then sums its x-side
  // partials in the same order, so the residual, the restart verdict, the PID
  // weight and ||A|| are bit-identical on all ranks (decisions cannot diverge
  // and desynchronise the collectives).
  Sched nside{};
  int grid_nside = 1;
  // Option B of SURVEY.md §8(e) ("sharded", the default at world > 1 without
  // the peer exchange; RHP_DIST_REPLICATED=1 keeps Option A): rank r owns
  // the column slice [nlo, nhi) = [r S, min((r+1) S, n)), S = ceil(n/P).
  // Per iteration: A_p^T y+_p (all n) is reduce-scattered to the owners,
  // the y-side sums of K1 and the x-side sums of the previous n-side walk go
  // through one 9-scalar allreduce, every rank runs the control on the same
  // sums, walks ONLY its slice (aty update + next primal step), and x+ is
  // all-gathered. Same bytes as the allreduce of Option A, n-side work 1/P.
  bool sharded = false;
  int64_t S = 0, nlo = 0, nhi = 0, nalloc = 0;  // nalloc = max(n, P S): padded n-vectors
  double* rsb = nullptr;   // [S] owned slice of the reduce-scattered A^T partial
  double* dsum = nullptr;  // [16] per-iteration scalars: y-side 0..4, x-side 5..8
  double* ksum = nullptr;  // [16] KKT scalars (row 0..3, col 4..9) / power dots (0..1)
  // CUDA graph of one block of iterations
  bool graph_built = false;
  cudaGraph_t graph = nullptr;
  cudaGraphExec_t gexec = nullptr;
  cudaEvent_t ev0 = nullptr, ev1 = nullptr, tev0 = nullptr, tev1 = nullptr;
  double last_block_ms = 0.0;
  int64_t host_total = 0;  // mirror of ctl->total after the last block
  int64_t host_check_interval = 64, host_iteration_limit = INT64_MAX;
  std::vector<double> hbuf;  // host scratch
  // row-partitioned multi-GPU
  bool dist = false;
  int rank = 0, world = 1;
  std::vector<int64_t> offsets;  // world+1 row offsets of the partition
  int64_t max_local = 0;         // largest local row count
  double* xchg = nullptr;        // [n + 16]: A_p^T partial | scalar sums (allreduced)
  // peer-memory exchange (peer.cuh, RHP_PEER_EXCHANGE=1): xchg then lives in
  // an IPC-shared region; peers' regions are opened at create
  bool peer = false;
  PeerView peerv{};
  std::vector<void*> peer_opened;
  unsigned int* peer_ticket = nullptr;
  double* ypad = nullptr;        // [max_local]
  double* ygather = nullptr;     // [world * max_local]
  int64_t* agree = nullptr;      // 1 int64 for host-decision agreement
  // small-LP cluster-resident blocks (resident.cuh)
  bool resident = false;
  int res_ctas = 1, res_wa = 1, res_wat = 1;
  size_t res_smem = 0;
  int32_t *res_a_split = nullptr, *res_at_split = nullptr;
  bool pdl = false;  // programmatic dependent launch of the SpMVs (launch_spmv, RHP_PDL=1)
  bool scaled = false;  // rhp_scale ran (it consumes the original values: once per ctx)
  // bounds that are one value on every row / column after scaling (bit 0
  // var_lb, 1 var_ub, 2 con_lb, 3 con_ub) and those values: the epilogues
  // take them from kernel parameters instead of loading them (ConstInputs)
  unsigned const_mask = 0;
  double const_val[4] = {0, 0, 0, 0};
  // per-operation API scratch (rhp_op_pdhg), allocated on first use:
  // 12 n-vectors then 11 m-vectors
  double* opbuf = nullptr;
  // rhp_set_csc_values(.., 1): the input's own CSC values as the source of
  // the A^T apply in rhp_scale (a matrix whose CSC values were produced by an
  // earlier scaling differs from its CSR values in the last ulp)
  double* csc_src = nullptr;
  // collectives of the partitioned path (comm.cuh): NCCL or an in-process group
  std::unique_ptr<Comm> comm;
  // plain-mode partitioned blocks: per-iteration stop flags written by
  // k_dist_control into mapped pinned memory, polled a few iterations behind
  // the launches so no collective is issued far past an on-device stop
  int* stop_mirror = nullptr;       // host pointer [block_limit]
  int* stop_mirror_dev = nullptr;   // its device alias
  std::vector<cudaEvent_t> it_events;
};

namespace {

// Uploads the warp schedule of an operator (built for the operator's grid).
void upload_sched(DevOp& d, const HostOperator& h, cudaStream_t s) {
  const size_t W = static_cast<size_t>(h.sched.n_chunks), ns = h.slot_row.size();
  d.warp_row = dev_alloc<int64_t>(W + 1);
  d.warp_nz = dev_alloc<int64_t>(W + 1);
  d.head_slot = dev_alloc<int32_t>(W);
  d.tail_slot = dev_alloc<int32_t>(W);
  d.slot_part = dev_alloc<double>(2 * W);
  upload(d.warp_row, h.warp_row.data(), W + 1, s);
  upload(d.warp_nz, h.warp_nz.data(), W + 1, s);
  upload(d.head_slot, h.head_slot.data(), W, s);
  upload(d.tail_slot, h.tail_slot.data(), W, s);
  d.slot_row = dev_alloc<int64_t>(ns);
  d.slot_first = dev_alloc<int32_t>(ns);
  d.slot_count = dev_alloc<int32_t>(ns);
  upload(d.slot_row, h.slot_row.data(), ns, s);
  upload(d.slot_first, h.slot_first.data(), ns, s);
  upload(d.slot_count, h.slot_count.data(), ns, s);
  d.slot_ticket = dev_alloc<unsigned int>(std::max<size_t>(ns, 1));  // zeroed by dev_alloc
  d.long_red = dev_alloc<double>(std::max<size_t>(ns, 1) * 16);
  d.sched = h.sched;
  d.sched.rp = d.rp;
  d.sched.warp_row = d.warp_row;
  d.sched.warp_nz = d.warp_nz;
  d.sched.head_slot = d.head_slot;
  d.sched.tail_slot = d.tail_slot;
  d.sched.slot_row = d.slot_row;
  d.sched.slot_first = d.slot_first;
  d.sched.slot_count = d.slot_count;
  d.sched.slot_part = d.slot_part;
  d.sched.slot_ticket = d.slot_ticket;
  d.sched.long_red = d.long_red;
  CK(cudaStreamSynchronize(s));
}

void free_op(DevOp& d) {
  for (DevOp& g : d.segs) free_op(g);
  for (void* p : {(void*)d.rp, (void*)d.ci, (void*)d.v, (void*)d.v_orig, (void*)d.warp_row,
                  (void*)d.warp_nz, (void*)d.slot_row, (void*)d.head_slot, (void*)d.tail_slot,
                  (void*)d.slot_first, (void*)d.slot_count, (void*)d.slot_part,
                  (void*)d.long_red, (void*)d.slot_ticket, (void*)d.segbuf, (void*)d.cta_row,
                  (void*)d.sell_ci, (void*)d.sell_v})
    if (p) cudaFree(p);
  d = DevOp{};
}

// The operator whose schedule carries the fused epilogue: the last column
// segment of a segmented operator, else the operator itself. K3 and the
// partitioned walkers walk its schedule and K1's finalize reads its slots.
const DevOp& fin(const DevOp& op) { return op.segs.empty() ? op : op.segs.back(); }

// The map of the n-side walkers and of the x-side partials (part3 layout):
// single GPU: A^T's schedule (K3 bit-identical to K2's fused primal step);
// row-partitioned: the rank-independent column map (rhp_ctx::nside).
const Sched& nside_sched(const rhp_ctx& c);
int nside_grid(const rhp_ctx& c);
const double* nside_long_red(const rhp_ctx& c);

// First index of a contiguous ascending permutation (the layout keeps rows
// and columns in their original order, so every map is one), else -1.
int64_t contiguous_start(const std::vector<int32_t>& perm) {
  for (size_t i = 1; i < perm.size(); ++i)
    if (perm[i] != perm[i - 1] + 1) return -1;
  return perm.empty() ? 0 : perm[0];
}

// Host loop over [0, n) split across the host's threads (the order maps of a
// relabelled layout touch tens of millions of entries per vector copy).
template <class F>
void host_parallel_for(size_t n, F&& f) {
  const size_t hw = std::max(1u, std::thread::hardware_concurrency());
  const size_t T = std::min<size_t>(std::min<size_t>(hw, 16), n / (1u << 20) + 1);
  if (T <= 1) {
    f(size_t{0}, n);
    return;
  }
  std::vector<std::thread> th;
  th.reserve(T);
  for (size_t t = 0; t < T; ++t) th.emplace_back([&, t] { f(n * t / T, n * (t + 1) / T); });
  for (auto& x : th) x.join();
}

// gather a host vector in original order into device order
void upload_perm(double* dst, const double* src, const std::vector<int32_t>& perm,
                 std::vector<double>& scratch, cudaStream_t s) {
  const int64_t start = contiguous_start(perm);
  if (start >= 0) {
    upload(dst, src + start, perm.size(), s);
    CK(cudaStreamSynchronize(s));
    return;
  }
  scratch.resize(perm.size());
  host_parallel_for(perm.size(), [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) scratch[i] = src[perm[i]];
  });
  upload(dst, scratch.data(), scratch.size(), s);
  CK(cudaStreamSynchronize(s));  // scratch is reused
}

void download_perm(double* dst, const double* src_dev, const std::vector<int32_t>& perm,
                   std::vector<double>& scratch, cudaStream_t s) {
  const int64_t start = contiguous_start(perm);
  if (start >= 0) {
    if (!perm.empty())
      CK(cudaMemcpyAsync(dst + start, src_dev, perm.size() * sizeof(double), cudaMemcpyDeviceToHost, s));
    CK(cudaStreamSynchronize(s));
    return;
  }
  scratch.resize(perm.size());
  if (!perm.empty())
    CK(cudaMemcpyAsync(scratch.data(), src_dev, perm.size() * sizeof(double),
                       cudaMemcpyDeviceToHost, s));
  CK(cudaStreamSynchronize(s));
  host_parallel_for(perm.size(), [&](size_t lo, size_t hi) {
    for (size_t i = lo; i < hi; ++i) dst[perm[i]] = scratch[i];
  });
}

// perm for local rows: prow holds global row ids; make them local
std::vector<int32_t> local_rows(const rhp_ctx& c) {
  std::vector<int32_t> p(c.L.prow.size());
  for (size_t i = 0; i < p.size(); ++i) p[i] = static_cast<int32_t>(c.L.prow[i] - c.L.row_begin);
  return p;
}

int vec_grid(const rhp_ctx& c, int64_t len) {
  const int64_t need = (len + kBlock - 1) / kBlock;
  return static_cast<int>(std::max<int64_t>(1, std::min<int64_t>(need, (int64_t)c.sm_count * 8)));
}

// With RHP_PDL=1 every SpMV is launched with programmatic stream
// serialization: spmv_fused waits for its predecessor with
// griddepcontrol.wait, so its launch and CTA rasterisation overlap the
// predecessor's tail. Off by default: measured inside the block graph it
// gains nothing on C2 (6904 vs 6895 iter/s) and loses 6% on C3 (20.1k vs
// 18.9k) — the graph already launches the next kernel back to back.
template <class Epi>
void launch_one(rhp_ctx& c, const DevOp& op, int grid, const double* xg, const Epi& epi,
                double* part, unsigned int* ticket, cudaStream_t s) {
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(grid));
  cfg.blockDim = dim3(kBlock);
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = c.pdl ? 1 : 0;
  if (op.cta_row) {
    const int32_t* cr = op.cta_row;
    cfg.gridDim = dim3(static_cast<unsigned>(op.cta_grid));
    if (op.l1g) CK(cudaLaunchKernelEx(&cfg, spmv_cta_rows<Epi, true>, op.csr(), xg, op.sched, cr, epi, part, ticket));
    else CK(cudaLaunchKernelEx(&cfg, spmv_cta_rows<Epi, false>, op.csr(), xg, op.sched, cr, epi, part, ticket));
    return;
  }
  if (op.sched.thread_rows) {
    if (op.l1g) CK(cudaLaunchKernelEx(&cfg, spmv_rows<Epi, true>, op.csr(), xg, op.sched, epi, part, ticket));
    else CK(cudaLaunchKernelEx(&cfg, spmv_rows<Epi, false>, op.csr(), xg, op.sched, epi, part, ticket));
    return;
  }
  if (op.l1g) CK(cudaLaunchKernelEx(&cfg, spmv_fused<Epi, true>, op.csr(), xg, op.sched, epi, part, ticket));
  else CK(cudaLaunchKernelEx(&cfg, spmv_fused<Epi, false>, op.csr(), xg, op.sched, epi, part, ticket));
}

EpiStore store_into(double* out);

// One SpMV with its fused epilogue; a column-segmented operator runs its
// segments in order (each adds its row sums to segbuf), the last one with
// the epilogue.
template <class Epi>
void launch_spmv(rhp_ctx& c, const DevOp& op, int grid, const double* xg, const Epi& epi,
                 double* part, unsigned int* ticket, cudaStream_t s) {
  if (op.segs.empty()) {
    launch_one(c, op, grid, xg, epi, part, ticket, s);
    return;
  }
  EpiSegStore<Epi> seg{};
  seg.gate = epi;
  for (size_t k = 0; k + 1 < op.segs.size(); ++k) {
    seg.out = op.segs[k].seg_out;
    launch_one(c, op.segs[k], grid, xg, seg, nullptr, nullptr, s);
  }
  launch_one(c, op.segs.back(), grid, xg, epi, part, ticket, s);
}

// Resident CTAs per SM of the thread-per-row kernel of an epilogue.
template <class Epi>
int prepare_rows() {
  int b = 0, b1 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &b, reinterpret_cast<const void*>(spmv_rows<Epi, false>), kBlock, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &b1, reinterpret_cast<const void*>(spmv_rows<Epi, true>), kBlock, 0));
  b = std::min(b, b1);
  if (b < 1) throw CudaError("spmv kernel does not fit on an SM");
  return b;
}

// Resident CTAs per SM of an SpMV instantiation.
template <class Epi>
int prepare_spmv() {
  int b = 0, b1 = 0;
  const size_t dyn = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &b, reinterpret_cast<const void*>(spmv_fused<Epi, false>), kBlock, dyn));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &b1, reinterpret_cast<const void*>(spmv_fused<Epi, true>), kBlock, dyn));
  b = std::min(b, b1);
  for (const void* fn : {reinterpret_cast<const void*>(spmv_rows<Epi, false>),
                         reinterpret_cast<const void*>(spmv_rows<Epi, true>)}) {
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&b1, fn, kBlock, dyn));
    b = std::min(b, b1);
  }
  if (b < 1) throw CudaError("spmv kernel does not fit on an SM");
  return b;
}

PrimalOut primal_out(rhp_ctx& c) { return PrimalOut{c.x, c.xp}; }

// Marks epilogue input k constant when bound `which` (0 vl, 1 vu, 2 cl, 3 cu)
// is constant (rhp_ctx::const_mask).
void mark_const(const rhp_ctx& c, ConstInputs& ci, int k, int which) {
  if ((c.const_mask >> which) & 1u) {
    ci.mask |= 1u << k;
    ci.val[k] = c.const_val[which];
  }
}

// rhp_ctx::const_mask of the final (scaled) bounds; RHP_CONST_INPUTS=0
// disables it (A/B). Decided per rank from its own vectors: it only selects
// where a value is read from, never the value.
void detect_constant_inputs(rhp_ctx& c) {
  c.const_mask = 0;
  if (const char* e = std::getenv("RHP_CONST_INPUTS"); e && std::atoi(e) == 0) return;
  const double* vec[4] = {c.vl, c.vu, c.cl, c.cu};
  const int64_t len[4] = {c.n, c.n, c.m, c.m};
  unsigned* flags = dev_alloc<unsigned>(4);
  CK(cudaMemsetAsync(flags, 0, 4 * sizeof(unsigned), c.stream));
  for (int q = 0; q < 4; ++q)
    if (len[q] > 0)
      k_not_constant<<<vec_grid(c, len[q]), kBlock, 0, c.stream>>>(vec[q], len[q], flags + q);
  CK(cudaGetLastError());
  unsigned h[4];
  CK(cudaMemcpyAsync(h, flags, sizeof(h), cudaMemcpyDeviceToHost, c.stream));
  for (int q = 0; q < 4; ++q)
    if (len[q] > 0)
      CK(cudaMemcpyAsync(&c.const_val[q], vec[q], sizeof(double), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  CK(cudaFree(flags));
  for (int q = 0; q < 4; ++q)
    if (len[q] > 0 && h[q] == 0) c.const_mask |= 1u << q;
}

EpiStore store_into(double* out) {
  EpiStore e{};
  e.out = out;
  return e;
}

// Gather-ceiling probe: the irreducible work of one SpMV over an operator's
// own nonzeros — stream its column indices and values coalesced, gather
// x[col] (8-B loads through the operator's cache policy), one FMA each — at
// full occupancy, with no rows, scans or epilogue. No SpMV over that operator
// can beat it, so bench.py reports K1/K2 against it next to the HBM roofline.
template <bool L1G>
__global__ void __launch_bounds__(256) k_gather_probe(const int32_t* __restrict__ ci,
                                                      const double* __restrict__ v,
                                                      const double* __restrict__ x, int64_t nnz,
                                                      double* out) {
  constexpr int U = 4;
  double s = 0.0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x * U;
  for (int64_t b = static_cast<int64_t>(blockIdx.x) * blockDim.x * U + threadIdx.x; b < nnz; b += stride) {
    int c[U];
    double w[U];
#pragma unroll
    for (int k = 0; k < U; ++k) {
      const int64_t i = b + static_cast<int64_t>(k) * blockDim.x;
      c[k] = i < nnz ? __ldcs(ci + i) : 0;
      w[k] = i < nnz ? __ldcs(v + i) : 0.0;
    }
    double g[U];
#pragma unroll
    for (int k = 0; k < U; ++k) g[k] = ld_gather<L1G>(x + c[k]);
#pragma unroll
    for (int k = 0; k < U; ++k) s = fma(w[k], g[k], s);
  }
  out[static_cast<size_t>(blockIdx.x) * blockDim.x + threadIdx.x] = s;
}

// SpMV engine per operator (deterministic, from the row lengths only, so two
// contexts on one LP always agree bit for bit): thread-per-row when the
// longest row has <= kThreadRowMax nonzeros, else the merge-path warp engine.
// RHP_THREAD_ROWS=0 forces merge path; =1 allows rows up to 64 nonzeros.
bool thread_rows_rule(const std::vector<int64_t>& rp, int64_t* longest_out = nullptr) {
  // RHP_THREAD_ROWS: 0 forces the merge path, 1 allows rows up to 64, a
  // larger number is the cap itself (A/B runs)
  const char* env = std::getenv("RHP_THREAD_ROWS");
  int64_t cap = kThreadRowMax;
  if (env) {
    const long v = std::atol(env);
    cap = v == 0 ? -1 : v == 1 ? 64 : v;
  }
  const int64_t rows = static_cast<int64_t>(rp.size()) - 1;
  int64_t longest = 0;
  for (int64_t r = 0; r < rows; ++r) longest = std::max(longest, rp[r + 1] - rp[r]);
  if (longest_out) *longest_out = longest;
  return rows > 0 && longest <= cap;
}

void apply_engine_rule(DevOp& d, const std::vector<int64_t>& rp) {
  const int64_t rows = static_cast<int64_t>(rp.size()) - 1;
  int64_t longest = 0;
  if (thread_rows_rule(rp, &longest)) {
    d.sched.thread_rows = 1;
    d.sched.n_multi = 0;  // no split rows: K1's finalize reads no slots of this operator
    // every row of one length: row starts are arithmetic (RHP_UNIFORM=0 off)
    const char* u = std::getenv("RHP_UNIFORM");
    if (rp[0] == 0 && rp[rows] == rows * longest && longest > 0 && (!u || std::atoi(u) != 0) &&
        rp[rows] <= INT64_MAX / 32)
      d.sched.uniform_len = static_cast<int32_t>(longest);
  }
}

// Long-row engine (spmv.cuh spmv_cta_rows) for an operator whose every row
// has >= kCtaRowMin nonzeros (C3's A: 2000 rows of 1000): CTA row runs
// balanced by nonzeros over the operator's grid. Only for A — A^T's
// schedule is also walked by K3 / the partitioned walkers, which need the
// merge-path or thread-per-row map. RHP_CTA_ROWS=0 disables it.
void apply_cta_rule(rhp_ctx& c, DevOp& d, const std::vector<int64_t>& rp) {
  const char* env = std::getenv("RHP_CTA_ROWS");
  if (env && env[0] == '0') return;
  const int64_t rows = static_cast<int64_t>(rp.size()) - 1;
  if (rows < 1 || rows > INT32_MAX) return;
  for (int64_t r = 0; r < rows; ++r)
    if (rp[r + 1] - rp[r] < kCtaRowMin) return;
  // as many CTAs as fit resident (all of them at once), at most one per row,
  // never more than the partial buffers hold
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
      &occ, reinterpret_cast<const void*>(spmv_cta_rows<EpiDual, false>), kBlock, 0));
  const int grid = static_cast<int>(std::max<int64_t>(
      1, std::min<int64_t>({rows, static_cast<int64_t>(c.sm_count) * std::max(occ, 1),
                            static_cast<int64_t>(c.grid_max)})));
  std::vector<int32_t> cr(static_cast<size_t>(grid) + 1, static_cast<int32_t>(rows));
  cr[0] = 0;
  const double total = static_cast<double>(rp[rows]);
  int64_t r = 0;
  for (int b = 1; b < grid; ++b) {
    const double goal = total * b / grid;
    while (r < rows && static_cast<double>(rp[r]) < goal) ++r;
    cr[b] = static_cast<int32_t>(r);
  }
  d.cta_row = dev_alloc<int32_t>(cr.size());
  d.cta_grid = grid;
  upload(d.cta_row, cr.data(), cr.size(), c.stream);
  CK(cudaStreamSynchronize(c.stream));
  d.sched.thread_rows = 0;
  d.sched.n_multi = 0;  // no split rows: K1's finalize reads no slots of this operator
}

// Sliced copy of an unsegmented uniform-length thread-per-row operator's
// (final, scaled) values: 32-row slices, element-major (Sched::sell_ci).
// Same elements, same order per row: bit-identical row sums. Off unless
// RHP_SLICED=1 — measured slower than CSR order.
void build_sliced(rhp_ctx& c, DevOp& d, bool always = false) {
  const char* e = std::getenv("RHP_SLICED");
  if (!always && (!e || std::atoi(e) == 0)) return;
  if (!d.segs.empty() || !d.sched.thread_rows || d.sched.uniform_len <= 0 || d.nnz == 0) return;
  const int64_t rows = d.rows, w = d.sched.uniform_len;
  const size_t cap = static_cast<size_t>((rows + 31) / 32 * 32 * w);
  d.sell_ci = dev_alloc<int32_t>(cap);
  d.sell_v = dev_alloc<double>(cap);
  k_build_sliced<<<vec_grid(c, rows), kBlock, 0, c.stream>>>(d.ci, d.v, rows, static_cast<int>(w),
                                                              d.sell_ci, d.sell_v);
  CK(cudaGetLastError());
  CK(cudaStreamSynchronize(c.stream));
  d.sched.sell_ci = d.sell_ci;
  d.sched.sell_v = d.sell_v;
}

// Thread-per-row row band (round 2). A merge-path operator may hold a long
// run of rows of one length w in (kThreadRowMax, 64] whose columns advance
// with the row at every element position (C4's arc-capacity rows: row e
// holds x[k*E + e] for the 25 commodities k, so rows e..e+31 read
// x[k*E + e .. e+31] at element k). Walked one row per thread, a warp's
// gathers of one element position are then one or two 128-B lines instead
// of 32 scattered sectors. Such a band is carved out of the final pass into
// its own segment (thread-per-row, uniform rows, sums stored to segbuf like
// a column segment's) and the final pass sees those rows as empty and adds
// their sums. A band's row sums are sequential in element order (the
// reference's order). Taken when the band holds >= 5 % of the nonzeros and
// >= 4096 rows, lies outside the column-segment band, and a sample of
// 32-row slices touches <= 12 distinct 32-B sectors per element position
// (8 for 32 consecutive doubles; random columns touch ~32). RHP_ROW_BAND=0 disables it, =force
// skips the size and sector tests (tests).
void carve_row_band(rhp_ctx& c, DevOp& d, int64_t cols, int grid) {
  const char* env = std::getenv("RHP_ROW_BAND");
  if (env && env[0] == '0') return;
  const bool force = env && std::strcmp(env, "force") == 0;
  if (d.cta_row || d.rows < 32) return;
  const bool had_segs = !d.segs.empty();
  const DevOp& f = had_segs ? d.segs.back() : d;
  if (f.sched.thread_rows || f.nnz == 0) return;
  const int64_t rows = f.rows;
  std::vector<int64_t> rp(static_cast<size_t>(rows) + 1);
  CK(cudaMemcpyAsync(rp.data(), f.rp, rp.size() * sizeof(int64_t), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
  // the longest run (by nonzeros) of equal-length rows with kThreadRowMax < w <= 64,
  // outside the column-segment band
  int64_t rb = -1, re = -1, w = 0, best = 0;
  for (int64_t i = 0; i < rows;) {
    const int64_t L = rp[i + 1] - rp[i];
    int64_t j = i + 1;
    while (j < rows && rp[j + 1] - rp[j] == L) ++j;
    int64_t a = i, b = j;
    if (had_segs && a < d.seg_re && b > d.seg_rb) {  // keep the part outside [seg_rb, seg_re)
      if (a >= d.seg_rb) a = std::max(a, d.seg_re);
      else b = std::min(b, d.seg_rb);
    }
    if (L > kThreadRowMax && L <= 64 && b > a && (b - a) * L > best) {
      best = (b - a) * L;
      rb = a;
      re = b;
      w = L;
    }
    i = j;
  }
  if (rb < 0 || re - rb < 32) return;
  if (!force && (re - rb < 4096 || static_cast<double>(best) < 0.05 * static_cast<double>(f.nnz)))
    return;
  if (!force) {  // sectors per element position over sampled 32-row slices
    const int64_t slices = (re - rb) / 32, samples = std::min<int64_t>(64, slices);
    std::vector<int32_t> buf(static_cast<size_t>(32 * w));
    double sectors = 0.0;
    for (int64_t k = 0; k < samples; ++k) {
      const int64_t r0 = rb + 32 * (slices * k / samples);
      CK(cudaMemcpyAsync(buf.data(), f.ci + rp[r0], buf.size() * sizeof(int32_t),
                         cudaMemcpyDeviceToHost, c.stream));
      CK(cudaStreamSynchronize(c.stream));
      for (int64_t t = 0; t < w; ++t) {
        int32_t sec[32];
        for (int r = 0; r < 32; ++r) sec[r] = buf[static_cast<size_t>(r * w + t)] >> 2;
        std::sort(sec, sec + 32);
        sectors += static_cast<double>(std::unique(sec, sec + 32) - sec);
      }
    }
    if (sectors / static_cast<double>(samples * w) > 12.0) return;
  }
  const int64_t eb = rp[rb], ee = rp[re], nb = re - rb;
  // the band: its rows with all their elements (uniform rows)
  DevOp band;
  band.rows = nb;
  band.nnz = ee - eb;
  band.rp = dev_alloc<int64_t>(static_cast<size_t>(nb) + 1);
  band.ci = dev_alloc<int32_t>(static_cast<size_t>(band.nnz));
  band.v = dev_alloc<double>(static_cast<size_t>(band.nnz));
  HostOperator hb;
  hb.rows = nb;
  hb.nnz = band.nnz;
  hb.rp.resize(static_cast<size_t>(nb) + 1);
  for (int64_t r = 0; r <= nb; ++r) hb.rp[r] = r * w;
  upload(band.rp, hb.rp.data(), hb.rp.size(), c.stream);
  CK(cudaMemcpyAsync(band.ci, f.ci + eb, band.nnz * sizeof(int32_t), cudaMemcpyDeviceToDevice, c.stream));
  CK(cudaMemcpyAsync(band.v, f.v + eb, band.nnz * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  // the final pass: every row, the band's rows empty
  DevOp fin2;
  fin2.rows = rows;
  fin2.nnz = f.nnz - band.nnz;
  HostOperator hf;
  hf.rows = rows;
  hf.nnz = fin2.nnz;
  hf.rp.resize(static_cast<size_t>(rows) + 1);
  for (int64_t r = 0; r <= rows; ++r) hf.rp[r] = r <= rb ? rp[r] : r <= re ? eb : rp[r] - (ee - eb);
  fin2.rp = dev_alloc<int64_t>(static_cast<size_t>(rows) + 1);
  fin2.ci = dev_alloc<int32_t>(static_cast<size_t>(fin2.nnz));
  fin2.v = dev_alloc<double>(static_cast<size_t>(fin2.nnz));
  upload(fin2.rp, hf.rp.data(), hf.rp.size(), c.stream);
  CK(cudaMemcpyAsync(fin2.ci, f.ci, eb * sizeof(int32_t), cudaMemcpyDeviceToDevice, c.stream));
  CK(cudaMemcpyAsync(fin2.v, f.v, eb * sizeof(double), cudaMemcpyDeviceToDevice, c.stream));
  CK(cudaMemcpyAsync(fin2.ci + eb, f.ci + ee, (f.nnz - ee) * sizeof(int32_t), cudaMemcpyDeviceToDevice,
                     c.stream));
  CK(cudaMemcpyAsync(fin2.v + eb, f.v + ee, (f.nnz - ee) * sizeof(double), cudaMemcpyDeviceToDevice,
                     c.stream));
  CK(cudaStreamSynchronize(c.stream));
  hb.cols = hf.cols = cols;
  for (HostOperator* h : {&hb, &hf}) build_schedule(*h, static_cast<int64_t>(grid) * kWarps, kRowWeight);
  upload_sched(band, hb, c.stream);
  upload_sched(fin2, hf, c.stream);
  band.sched.thread_rows = 1;
  band.sched.n_multi = 0;
  band.sched.uniform_len = static_cast<int32_t>(w);
  apply_engine_rule(fin2, hf.rp);
  band.l1g = fin2.l1g = d.l1g;
  if (!d.segbuf) d.segbuf = dev_alloc<double>(static_cast<size_t>(d.rows));
  band.sched.seg_in = nullptr;  // the band's first and only partial sums
  band.seg_out = d.segbuf + rb;
  fin2.sched.seg_in = d.segbuf;
  band.seg_rb = rb;
  band.seg_re = re;
  // element-major slices: a warp's loads of one element position of its 32
  // rows are one line of indices and two of values (row-major, 25-element
  // rows put every lane on its own lines: K1 679 -> 747 us on C4)
  if (!(std::getenv("RHP_ROW_BAND_CSR"))) build_sliced(c, band, true);
  if (had_segs) {
    free_op(d.segs.back());
    d.segs.back() = fin2;
    d.segs.insert(d.segs.end() - 1, band);
  } else {
    d.segs.push_back(band);
    d.segs.push_back(fin2);
  }
  d.row_band = true;
}

void choose_engines(rhp_ctx& c) {
  apply_engine_rule(c.A, c.L.A.rp);
  apply_engine_rule(c.At, c.L.At.rp);
  apply_cta_rule(c, c.A, c.L.A.rp);
}

__global__ void k_mark_sectors(const int32_t* ci, int64_t lo, int64_t hi, unsigned int* bits) {
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t e = lo + static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; e < hi; e += stride) {
    const uint32_t sector = static_cast<uint32_t>(ci[e]) >> 2;  // 4 doubles per 32-B sector
    atomicOr(bits + (sector >> 5), 1u << (sector & 31));
  }
}

__global__ void k_popcount(const unsigned int* bits, int64_t words, unsigned long long* total) {
  unsigned long long t = 0;
  const int64_t stride = static_cast<int64_t>(gridDim.x) * blockDim.x;
  for (int64_t i = static_cast<int64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < words; i += stride)
    t += __popc(bits[i]);
  if (t) atomicAdd(total, t);
}

// Gather footprint of the interleaved schedule (layout.cu: the grid walks
// one band of W consecutive chunks at a time): the distinct 32-B sectors of
// the gathered vector touched by a band, times 32 B, maximised over up to 8
// bands spread over the operator. Deterministic (structure only).
// Gather footprint of the bands of an operator: band b = the W consecutive
// merge-path chunks the whole grid walks at once (chunks bW .. bW+W-1), its
// footprint = distinct 32-B sectors of the gathered vector its nonzeros
// touch. Bands whose footprint exceeds `limit` gather mostly from DRAM. Up to
// 256 bands are measured (evenly spaced when there are more); the hull of
// the rows of the bad bands (each measured band standing for the rows up to
// its measured neighbours) is returned in [rb, re). False if none is bad.
bool bad_band_hull(rhp_ctx& c, const DevOp& d, const HostOperator& h, int64_t cols, double limit,
                   int64_t* rb, int64_t* re) {
  const int64_t W = h.sched.n_warps, chunks = h.sched.n_chunks, rows = h.rows;
  *rb = 0;
  *re = rows;
  if (W <= 0 || chunks <= W) return static_cast<double>(cols) * 8.0 > limit;  // one band
  const int64_t bands = chunks / W;
  const int64_t words = (cols / 4) / 32 + 2;
  unsigned int* bits = dev_alloc<unsigned int>(static_cast<size_t>(words));
  unsigned long long* total = dev_alloc<unsigned long long>(1);
  const int64_t samples = std::min<int64_t>(256, bands);
  std::vector<int64_t> band_of(static_cast<size_t>(samples));
  std::vector<char> bad(static_cast<size_t>(samples), 0);
  auto band_row = [&](int64_t b) { return h.warp_row[std::min(chunks, b * W)]; };
  for (int64_t k = 0; k < samples; ++k) {
    const int64_t b = bands * k / samples;
    band_of[k] = b;
    const int64_t lo = h.warp_nz[b * W], hi = h.warp_nz[std::min(chunks, (b + 1) * W)];
    CK(cudaMemsetAsync(bits, 0, words * sizeof(unsigned int), c.stream));
    CK(cudaMemsetAsync(total, 0, sizeof(unsigned long long), c.stream));
    if (hi > lo) k_mark_sectors<<<c.sm_count * 4, 256, 0, c.stream>>>(d.ci, lo, hi, bits);
    k_popcount<<<c.sm_count * 4, 256, 0, c.stream>>>(bits, words, total);
    unsigned long long t = 0;
    CK(cudaMemcpyAsync(&t, total, sizeof(t), cudaMemcpyDeviceToHost, c.stream));
    CK(cudaStreamSynchronize(c.stream));
    bad[k] = 32.0 * static_cast<double>(t) > limit;
  }
  cudaFree(bits);
  cudaFree(total);
  int64_t first = -1, last = -1;
  for (int64_t k = 0; k < samples; ++k)
    if (bad[k]) {
      if (first < 0) first = k;
      last = k;
    }
  if (first < 0) return false;
  *rb = first == 0 ? 0 : band_row(band_of[first - 1] + 1);
  *re = last == samples - 1 ? rows : band_row(band_of[last + 1]);
  if (*re <= *rb) {
    *rb = 0;
    *re = rows;
  }
  return true;
}

// Column segments (segments.cuh) of an operator whose gathered vector is
// larger than RHP_SEG_BYTES (default 64 MB, 0 disables) AND whose
// interleaved bands still gather from more than that (C5's random columns:
// yes; C4's commodity-ordered columns: no — there segments only add row
// passes, K1 0.39 -> 0.61 ms). RHP_SEG_FORCE=1 skips the band test (tests).
// Equal column ranges, each with its own merge-path schedule for the
// operator's grid and its own engine choice; the cache policy is the
// operator's. Built after scaling (the values are final), rebuilt if scaling
// runs again. A pure function of the structure, so it never makes two
// contexts on one LP differ.
void build_segments(rhp_ctx& c, DevOp& d, const HostOperator& h, int64_t cols, int grid) {
  for (DevOp& g : d.segs) free_op(g);
  d.segs.clear();
  if (d.segbuf) cudaFree(d.segbuf);
  d.segbuf = nullptr;
  double seg_bytes = 64.0 * 1024 * 1024;  // C5: 48 MB 68, 64 MB 74.8, 80 MB 66.8 iter/s
  if (const char* e = std::getenv("RHP_SEG_BYTES")) seg_bytes = std::atof(e);
  if (!(seg_bytes > 0) || d.nnz == 0 || d.cta_row) return;
  const int64_t S = static_cast<int64_t>(std::ceil(static_cast<double>(cols) * 8.0 / seg_bytes));
  if (S <= 1) return;
  const char* force = std::getenv("RHP_SEG_FORCE");
  int64_t rb = 0, re = d.rows;
  if (!(force && force[0] == '1') && !bad_band_hull(c, d, h, cols, seg_bytes, &rb, &re)) return;
  // RHP_SEG_BAND=0: split every row (the pre-band behaviour), for A/B runs;
  // RHP_SEG_BAND=<lo>,<hi>: that row band (tests, with RHP_SEG_FORCE=1)
  if (const char* e = std::getenv("RHP_SEG_BAND")) {
    long long lo = 0, hi = 0;
    if (std::sscanf(e, "%lld,%lld", &lo, &hi) == 2) {
      rb = std::max<int64_t>(0, std::min<int64_t>(lo, d.rows));
      re = std::max<int64_t>(rb, std::min<int64_t>(hi, d.rows));
    } else if (e[0] == '0') {
      rb = 0;
      re = d.rows;
    }
  }
  std::vector<int32_t> cb(static_cast<size_t>(S) + 1);
  for (int64_t k = 0; k <= S; ++k) cb[k] = static_cast<int32_t>(cols * k / S);
  std::vector<DeviceCsr> parts;
  std::vector<std::vector<int64_t>> hrp;
  split_columns(d, cb, rb, re, parts, hrp, c.stream);
  // running row sums: zero outside the band for good (only the band's rows
  // pass through the intermediate segments)
  d.segbuf = dev_alloc<double>(static_cast<size_t>(d.rows));
  d.seg_rb = rb;
  d.seg_re = re;
  d.segs.resize(static_cast<size_t>(S));
  for (int64_t k = 0; k < S; ++k) {
    DevOp& g = d.segs[k];
    const bool last = k == S - 1;
    static_cast<DeviceCsr&>(g) = parts[k];
    HostOperator hs;
    hs.rows = parts[k].rows;
    hs.cols = last ? cols : cb[k + 1] - cb[k];
    hs.nnz = parts[k].nnz;
    hs.rp = std::move(hrp[k]);
    build_schedule(hs, static_cast<int64_t>(grid) * kWarps, kRowWeight);
    upload_sched(g, hs, c.stream);
    apply_engine_rule(g, hs.rp);
    g.l1g = d.l1g;
    // intermediate segments read and write the band's slice of the running
    // sums (local row r -> segbuf[rb + r]); the last one reads every row's
    g.sched.seg_in = k == 0 ? nullptr : (last ? d.segbuf : d.segbuf + rb);
    g.seg_out = last ? nullptr : d.segbuf + rb;
  }
}

// Gather cache policy (ld_gather): L1::no_allocate, except A's gathers on a
// relabelled layout, which allocate in L1 (first-touch order puts a row's
// columns side by side, so neighbouring lanes and the next window re-read
// the lines: C4 K1 596 -> 586 us, 912 -> 929 iter/s, A/B twice on one box;
// Aᵀ neutral). Without relabelling L1 wins nowhere (C2 6958 vs 6620, C3
// 22.9k both, C4 1102 vs 1076 iter/s in round 1). RHP_L1_GATHER overrides:
// 0 none, 1 both operators, A / T one of them. Deterministic, and the policy
// never changes a result.
void choose_gather_policy(rhp_ctx& c) {
  const char* env = std::getenv("RHP_L1_GATHER");
  if (!env) {
    c.A.l1g = c.L.relabel;
    c.At.l1g = false;
    return;
  }
  c.A.l1g = env[0] == '1' || env[0] == 'A';
  c.At.l1g = env[0] == '1' || env[0] == 'T';
}

// Peer-memory exchange (peer.cuh): one cudaMalloc'd region per rank, its
// CUDA IPC handle all-gathered over the rank's NCCL communicator, the peers'
// regions opened and mapped. The local xchg moves into the region.
void setup_peers(rhp_ctx& c) {
#ifdef RHP_WITH_NCCL
  if (c.world > kMaxPeers) throw CudaError("peer exchange supports at most 16 ranks");
  const size_t n = static_cast<size_t>(c.n);
  const size_t doubles = (n + 16) + n + 8;
  const size_t bytes = doubles * sizeof(double) + 2 * kMaxPeers * sizeof(unsigned long long);
  void* region = nullptr;
  CK(cudaMalloc(&region, bytes));
  CK(cudaMemset(region, 0, bytes));
  cudaIpcMemHandle_t mine;
  CK(cudaIpcGetMemHandle(&mine, region));
  char* d_h = nullptr;
  CK(cudaMalloc(&d_h, sizeof(mine) * (c.world + 1)));
  CK(cudaMemcpy(d_h, &mine, sizeof(mine), cudaMemcpyHostToDevice));
  if (!c.comm->is_nccl()) throw CudaError("the peer-memory exchange needs the NCCL transport");
  c.comm->allgather(d_h, d_h + sizeof(mine), sizeof(mine), c.stream);
  std::vector<cudaIpcMemHandle_t> all(static_cast<size_t>(c.world));
  CK(cudaMemcpyAsync(all.data(), d_h + sizeof(mine), sizeof(mine) * c.world, cudaMemcpyDeviceToHost,
                     c.stream));
  CK(cudaStreamSynchronize(c.stream));
  CK(cudaFree(d_h));
  for (int q = 0; q < c.world; ++q) {
    void* ptr = region;
    if (q != c.rank) {
      CK(cudaIpcOpenMemHandle(&ptr, all[q], cudaIpcMemLazyEnablePeerAccess));
      c.peer_opened.push_back(ptr);
    }
    double* base = static_cast<double*>(ptr);
    c.peerv.xchg[q] = base;
    c.peerv.rbuf[q] = base + n + 16;
    c.peerv.flags[q] = reinterpret_cast<unsigned long long*>(base + doubles);
  }
  c.peerv.ysum = static_cast<double*>(region) + 2 * n + 16;
  c.peerv.rank = c.rank;
  c.peerv.world = c.world;
  c.peerv.n = c.n;
  if (c.xchg) CK(cudaFree(c.xchg));
  c.xchg = static_cast<double*>(region);
  c.peer_ticket = dev_alloc<unsigned int>(1);
  c.peer = true;
#else
  (void)c;
  throw CudaError("built without NCCL");
#endif
}

// (one rank keeps A^T's schedule: nothing to agree with, and the one-rank
// partitioned path stays bit-identical to the single-GPU path)
bool rank_independent_nside(const rhp_ctx& c) { return c.dist && c.world > 1; }
const Sched& nside_sched(const rhp_ctx& c) {
  return rank_independent_nside(c) ? c.nside : fin(c.At).sched;
}
int nside_grid(const rhp_ctx& c) { return rank_independent_nside(c) ? c.grid_nside : c.grid_at; }
const double* nside_long_red(const rhp_ctx& c) {
  return rank_independent_nside(c) ? nullptr : fin(c.At).long_red;
}

EpiDual epi_dual(rhp_ctx& c, int token) {
  EpiDual e{};
  e.ctl = c.ctl;
  e.y = c.y;
  e.ax = c.ax;
  e.yplus = c.yp;
  const double* in[] = {c.y, c.ax, c.cl, c.cu, c.y0, c.ax0};
  for (int k = 0; k < EpiDual::NIN; ++k) e.in[k] = in[k];
  mark_const(c, e.cin, 2, 2);
  mark_const(c, e.cin, 3, 3);
  e.part3 = c.part3;
  e.grid3 = nside_grid(c);
  e.n_multi3 = nside_sched(c).n_multi;
  e.long_red3 = nside_long_red(c);
  e.token = token;
  return e;
}

EpiAty epi_aty(rhp_ctx& c, int token) {
  EpiAty e{};
  e.ctl = c.ctl;
  e.aty = c.aty;
  e.o = primal_out(c);
  const double* in[] = {c.aty, c.aty0, c.x, c.c, c.vl, c.vu, c.x0};
  for (int k = 0; k < EpiAty::NIN; ++k) e.in[k] = in[k];
  mark_const(c, e.cin, 4, 0);
  mark_const(c, e.cin, 5, 1);
  e.token = token;
  return e;
}

void allreduce(rhp_ctx& c, double* buf, size_t count, cudaStream_t s) {
  c.comm->allreduce(buf, count, false, s);
}

void allreduce_max(rhp_ctx& c, double* buf, size_t count, cudaStream_t s) {
  c.comm->allreduce(buf, count, true, s);
}

void launch_iteration_sharded(rhp_ctx& c, int token, cudaStream_t s);

void launch_iteration(rhp_ctx& c, int token, cudaStream_t s, bool guard = false) {
  if (!c.dist) {
    EpiDual d = epi_dual(c, token);
    EpiAty a = epi_aty(c, token);
    d.guard = a.guard = guard ? 1 : 0;
    launch_spmv(c, c.A, c.grid_a, c.xp, d, c.part1, &c.ctl->ticket_dual, s);
    launch_spmv(c, c.At, c.grid_at, c.yp, a, c.part3, nullptr, s);
    return;
  }
  if (c.sharded) {
    launch_iteration_sharded(c, token, s);
    return;
  }
  // row-partitioned, Option A: local A x+ with the dual epilogue (y-side sums
  // -> xchg[n..]), local A_p^T y+_p -> xchg[0..n), one allreduce, control,
  // aty/primal epilogue over all n columns (replicated)
  EpiDual d = epi_dual(c, token);
  d.xchg = c.xchg + c.n;
  launch_spmv(c, c.A, c.grid_a, c.xp, d, c.part1, &c.ctl->ticket_dual, s);
  EpiStore st = store_into(c.xchg);
  st.ctl = c.ctl;
  st.token = token;
  launch_spmv(c, c.At, c.grid_at, c.yp, st, nullptr, nullptr, s);
  if (c.peer) {  // A^T y exchange over NVLink peer memory (peer.cuh)
    k_peer_signal<<<1, 32, 0, s>>>(c.ctl, token, c.peerv);
    k_peer_reduce<<<c.grid_vec, kBlock, 0, s>>>(c.ctl, token, c.peerv, c.peer_ticket);
    k_peer_gather<<<c.grid_vec, kBlock, 0, s>>>(c.ctl, token, c.peerv);
    CK(cudaGetLastError());
  } else {
    allreduce(c, c.xchg, static_cast<size_t>(c.n) + 5, s);
  }
  k_dist_control<<<1, kBlock, 0, s>>>(c.ctl, c.part3, nside_grid(c), nside_sched(c).n_multi,
                                      nside_long_red(c), c.xchg + c.n, token, nullptr);
  CK(cudaGetLastError());
  EpiAtyDist e{};
  e.ctl = c.ctl;
  e.aty = c.aty;
  e.o = primal_out(c);
  const double* in[] = {c.xchg, c.aty, c.aty0, c.x, c.c, c.vl, c.vu, c.x0};
  for (int k = 0; k < EpiAtyDist::NIN; ++k) e.in[k] = in[k];
  mark_const(c, e.cin, 5, 0);
  mark_const(c, e.cin, 6, 1);
  e.token = token;
  epilogue_walk<EpiAtyDist><<<nside_grid(c), kBlock, 0, s>>>(nside_sched(c), e, c.part3);
  CK(cudaGetLastError());
}

// Sharded n-side walk epilogue tail: this rank's x-side sums of the walk
// into dsum[5..9) (summed across ranks by the next iteration's allreduce),
// then every rank's x+ slice to every rank (in-place all-gather).
void sharded_walk_tail(rhp_ctx& c, cudaStream_t s) {
  k_sum_partials<4><<<1, kBlock, 0, s>>>(c.part3, c.grid_nside, c.dsum + 5);
  CK(cudaGetLastError());
  c.comm->allgather(c.xp + c.S * c.rank, c.xp, static_cast<size_t>(c.S) * sizeof(double), s);
}

// One iteration of the sharded partitioned path (Option B, rhp_ctx::sharded).
void launch_iteration_sharded(rhp_ctx& c, int token, cudaStream_t s) {
  const int64_t lo = c.nlo;
  EpiDual d = epi_dual(c, token);
  d.xchg = c.dsum;  // y-side sums -> dsum[0..5)
  launch_spmv(c, c.A, c.grid_a, c.xp, d, c.part1, &c.ctl->ticket_dual, s);
  EpiStore st = store_into(c.xchg);
  st.ctl = c.ctl;
  st.token = token;
  launch_spmv(c, c.At, c.grid_at, c.yp, st, nullptr, nullptr, s);
  c.comm->reduce_scatter(c.xchg, c.rsb, static_cast<size_t>(c.S), s);
  allreduce(c, c.dsum, 9, s);  // y-side (this iteration) + x-side (previous walk) sums
  k_dist_control<<<1, kBlock, 0, s>>>(c.ctl, c.part3, c.grid_nside, 0, nullptr, c.dsum, token,
                                      c.dsum + 5);
  CK(cudaGetLastError());
  EpiAtyDist e{};
  e.ctl = c.ctl;
  e.aty = c.aty + lo;
  e.o = PrimalOut{c.x + lo, c.xp + lo};
  const double* in[] = {c.rsb, c.aty + lo, c.aty0 + lo, c.x + lo, c.c + lo, c.vl + lo, c.vu + lo,
                        c.x0 + lo};
  for (int k = 0; k < EpiAtyDist::NIN; ++k) e.in[k] = in[k];
  mark_const(c, e.cin, 5, 0);
  mark_const(c, e.cin, 6, 1);
  e.token = token;
  epilogue_walk<EpiAtyDist><<<c.grid_nside, kBlock, 0, s>>>(c.nside, e, c.part3);
  CK(cudaGetLastError());
  sharded_walk_tail(c, s);
}

// Contiguous split of an operator's rows into `parts` runs balanced by
// nonzeros + rows.
std::vector<int32_t> split_rows(const std::vector<int64_t>& rp, int parts) {
  const int64_t rows = static_cast<int64_t>(rp.size()) - 1;
  std::vector<int32_t> s(static_cast<size_t>(parts) + 1, static_cast<int32_t>(rows));
  s[0] = 0;
  const double total = static_cast<double>(rp[rows] + rows);
  int p = 1;
  for (int64_t i = 0; i < rows && p < parts; ++i)
    if (static_cast<double>(rp[i + 1] + i + 1) >= total * p / parts) s[p++] = static_cast<int32_t>(i + 1);
  return s;
}

int lanes_for(int64_t nnz, int64_t rows) {
  const int64_t mean = rows > 0 ? (nnz + rows - 1) / rows : 1;
  return mean <= 4 ? 1 : mean <= 8 ? 2 : mean <= 16 ? 4 : mean <= 32 ? 8 : mean <= 64 ? 16 : 32;
}

// Shared-memory bytes of a CSR slice staged by the resident kernel.
size_t slice_bytes(const std::vector<int64_t>& rp, int32_t r0, int32_t r1) {
  const size_t rows = static_cast<size_t>(r1 - r0), nz = static_cast<size_t>(rp[r1] - rp[r0]);
  auto a16 = [](size_t x) { return (x + 15) & ~size_t(15); };
  return a16(4 * (rows + 1)) + a16(8 * nz) + a16(4 * nz);
}

// Chooses the cluster (up to 16 CTAs, one per SM) and row splits; false if
// the per-CTA matrix slices do not fit in shared memory.
bool setup_resident(rhp_ctx& c) {
  const void* fn = reinterpret_cast<const void*>(k_resident);
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeNonPortableClusterSizeAllowed, 1));
  CK(cudaFuncSetAttribute(fn, cudaFuncAttributeMaxDynamicSharedMemorySize,
                          static_cast<int>(kResSmemMax)));
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(kResMaxCtas);
  cfg.blockDim = dim3(kResThreads);
  cfg.dynamicSmemBytes = kResSmemMax;
  int max_cluster = 1;
  CK(cudaOccupancyMaxPotentialClusterSize(&max_cluster, fn, &cfg));
  // the smallest cluster of {8, 16} CTAs whose slices fit: fewer CTAs make
  // the two cluster barriers and the DSMEM reductions cheaper (C1: 16 CTAs
  // 112k, 8 CTAs 123k, 4 CTAs 90k iter/s); RHP_RES_CTAS caps the size
  int cap = std::max(1, std::min(kResMaxCtas, max_cluster));
  if (const char* e = std::getenv("RHP_RES_CTAS")) cap = std::max(1, std::min(cap, std::atoi(e)));
  int ctas = 0;
  std::vector<int32_t> sa, st;
  size_t need = 0;
  for (int cand : {std::min(8, cap), cap}) {
    sa = split_rows(c.L.A.rp, cand);
    st = split_rows(c.L.At.rp, cand);
    need = 0;
    for (int r = 0; r < cand; ++r)  // matrix slices + the shared-memory iterate slices
      need = std::max(need, slice_bytes(c.L.A.rp, sa[r], sa[r + 1]) +
                                slice_bytes(c.L.At.rp, st[r], st[r + 1]) +
                                8 * (6 * static_cast<size_t>(sa[r + 1] - sa[r]) +
                                     7 * static_cast<size_t>(st[r + 1] - st[r])));
    if (need <= kResSmemMax) {
      ctas = cand;
      break;
    }
  }
  if (ctas == 0) return false;
  c.res_ctas = ctas;
  c.res_smem = std::max<size_t>(need, 16);
  c.res_a_split = dev_alloc<int32_t>(sa.size());
  c.res_at_split = dev_alloc<int32_t>(st.size());
  upload(c.res_a_split, sa.data(), sa.size(), c.stream);
  upload(c.res_at_split, st.data(), st.size(), c.stream);
  CK(cudaStreamSynchronize(c.stream));
  c.res_wa = lanes_for(c.L.nnz, c.m);
  c.res_wat = lanes_for(c.L.nnz, c.n);
  return true;
}

void launch_resident(rhp_ctx& c, cudaStream_t s) {
  ResParams p{};
  p.A = c.A.csr();
  p.At = c.At.csr();
  p.xp = c.xp;
  p.yp = c.yp;
  p.a_split = c.res_a_split;
  p.at_split = c.res_at_split;
  p.wa = c.res_wa;
  p.wat = c.res_wat;
  p.dual = epi_dual(c, 0);
  p.aty = epi_aty(c, 0);
  p.primal.ctl = c.ctl;
  p.primal.o = primal_out(c);
  const double* in[] = {c.aty, c.x, c.c, c.vl, c.vu, c.x0};
  for (int k = 0; k < EpiPrimal::NIN; ++k) p.primal.in[k] = in[k];
  mark_const(c, p.primal.cin, 3, 0);
  mark_const(c, p.primal.cin, 4, 1);
  p.ctl = c.ctl;
  cudaLaunchConfig_t cfg{};
  cfg.gridDim = dim3(static_cast<unsigned>(c.res_ctas));
  cfg.blockDim = dim3(kResThreads);
  cfg.dynamicSmemBytes = c.res_smem;
  cfg.stream = s;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeClusterDimension;
  attr[0].val.clusterDim.x = static_cast<unsigned>(c.res_ctas);
  attr[0].val.clusterDim.y = 1;
  attr[0].val.clusterDim.z = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  CK(cudaLaunchKernelEx(&cfg, k_resident, p));
}

void launch_primal_init(rhp_ctx& c, cudaStream_t s) {
  const int64_t lo = c.sharded ? c.nlo : 0;  // sharded: the owned slice only
  EpiPrimal e{};
  e.ctl = c.ctl;
  e.o = PrimalOut{c.x + lo, c.xp + lo};
  const double* in[] = {c.aty + lo, c.x + lo, c.c + lo, c.vl + lo, c.vu + lo, c.x0 + lo};
  for (int k = 0; k < EpiPrimal::NIN; ++k) e.in[k] = in[k];
  mark_const(c, e.cin, 3, 0);
  mark_const(c, e.cin, 4, 1);
  epilogue_walk<EpiPrimal><<<nside_grid(c), kBlock, 0, s>>>(nside_sched(c), e, c.part3);
  CK(cudaGetLastError());
  if (c.sharded) sharded_walk_tail(c, s);
}

void build_graph(rhp_ctx& c) {
  cudaStream_t cap;
  CK(cudaStreamCreateWithFlags(&cap, cudaStreamNonBlocking));
  CK(cudaGraphCreate(&c.graph, 0));
  cudaGraphConditionalHandle h;
  CK(cudaGraphConditionalHandleCreate(&h, c.graph, 1u, cudaGraphCondAssignDefault));
  unsigned long long hv = static_cast<unsigned long long>(h);
  CK(cudaMemcpy(&c.ctl->cond_handle, &hv, sizeof(hv), cudaMemcpyHostToDevice));
  // node 1: the block's first primal step
  CK(cudaStreamBeginCaptureToGraph(cap, c.graph, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  launch_primal_init(c, cap);
  cudaGraph_t g1;
  CK(cudaStreamEndCapture(cap, &g1));
  size_t count = 0;
  CK(cudaGraphGetNodes(c.graph, nullptr, &count));
  std::vector<cudaGraphNode_t> nodes(count);
  CK(cudaGraphGetNodes(c.graph, nodes.data(), &count));
  if (count != 1) throw CudaError("unexpected node count after capturing primal_init");
  // node 2: WHILE(!stop) { K1 ; K2 }
  cudaGraphNodeParams cp{};
  cp.type = cudaGraphNodeTypeConditional;
  cp.conditional.handle = h;
  cp.conditional.type = cudaGraphCondTypeWhile;
  cp.conditional.size = 1;
  cudaGraphNode_t cond;
  CK(cudaGraphAddNode(&cond, c.graph, nodes.data(), 1, &cp));
  cudaGraph_t body = cp.conditional.phGraph_out[0];
  CK(cudaStreamBeginCaptureToGraph(cap, body, nullptr, nullptr, 0,
                                   cudaStreamCaptureModeThreadLocal));
  // the body runs kGraphUnroll iterations: one conditional evaluation (a
  // device-side relaunch of the body) per kGraphUnroll K1/K2 pairs; copies
  // after the first skip themselves once a K1 has stopped the block
  for (int j = 0; j < kGraphUnroll; ++j) launch_iteration(c, j, cap, j > 0);
  cudaGraph_t g2;
  CK(cudaStreamEndCapture(cap, &g2));
  CK(cudaGraphInstantiate(&c.gexec, c.graph, 0));
  CK(cudaStreamDestroy(cap));
  c.graph_built = true;
}

template <class T>
void set_ctl(rhp_ctx& c, size_t offset, const T& v) {
  CK(cudaMemcpyAsync(reinterpret_cast<char*>(c.ctl) + offset, &v, sizeof(T),
                     cudaMemcpyHostToDevice, c.stream));
  CK(cudaStreamSynchronize(c.stream));
}
#define SET_CTL(ctx, field, val) set_ctl(ctx, offsetof(Ctl, field), (val))

void pull_ctl(rhp_ctx& c) {
  CK(cudaMemcpyAsync(c.ctl_host, c.ctl, sizeof(Ctl), cudaMemcpyDeviceToHost, c.stream));
  CK(cudaStreamSynchronize(c.stream));
}

// KKT sums of (xbar, ybar) = (xs, ys) in scaled space; optional refresh of
// z's caches and output of the unscaled vectors.
void run_kkt(rhp_ctx& c, const double* xs, const double* ys, bool refresh, bool write_out,
             rhp_kkt_sums* out) {
  EpiKktRow er{};
  er.ax_refresh = refresh ? c.ax : nullptr;
  er.yout = write_out ? c.yout : nullptr;
  er.in[0] = ys;
  er.in[1] = c.rs;
  er.in[2] = c.clo;
  er.in[3] = c.cuo;
  if (!c.dist) launch_spmv(c, c.A, c.grid_a, xs, er, c.partA, nullptr, c.stream);
  EpiKktCol ec{};
  ec.ctl = c.ctl;
  ec.aty_refresh = refresh ? c.aty : nullptr;
  ec.in[0] = xs;
  ec.in[1] = c.cs;
  ec.in[2] = c.co;
  ec.in[3] = c.vlo;
  ec.in[4] = c.vuo;
  ec.xout = write_out ? c.xout : nullptr;
  ec.rcout = write_out ? c.rcout : nullptr;
  ec.part_row = c.partA;
  ec.grid_row = c.A.cta_row ? c.A.cta_grid : c.grid_a;  // the A-side kernel's grid
  ec.n_multi_row = fin(c.A).sched.n_multi;
  ec.long_red_row = fin(c.A).long_red;
  if (!c.dist) {
    launch_spmv(c, c.At, c.grid_at, ys, ec, c.partAt, &c.ctl->ticket_kkt, c.stream);
  } else if (c.sharded) {
    // Option B: x needs all its slices for A_p x; the column side runs on the
    // owned slice of the reduce-scattered A^T y; row (0..3) and column
    // (4..9) sums meet in one 10-scalar allreduce
    cudaStream_t s = c.stream;
    const int64_t lo = c.nlo;
    if (xs == c.x)
      c.comm->allgather(c.x + c.S * c.rank, c.x, static_cast<size_t>(c.S) * sizeof(double), s);
    EpiKktRowDist rd{};
    static_cast<EpiKktRow&>(rd) = er;
    rd.xsums = c.ksum;
    launch_spmv(c, c.A, c.grid_a, xs, rd, c.partA, &c.ctl->ticket_kkt, s);
    launch_spmv(c, c.At, c.grid_at, ys, store_into(c.xchg), nullptr, nullptr, s);
    c.comm->reduce_scatter(c.xchg, c.rsb, static_cast<size_t>(c.S), s);
    EpiKktColDist cd{};
    cd.col = ec;
    cd.col.aty_refresh = refresh ? c.aty + lo : nullptr;
    cd.col.xout = write_out ? c.xout + lo : nullptr;
    cd.col.rcout = write_out ? c.rcout + lo : nullptr;
    const double* in[] = {c.rsb, xs + lo, c.cs + lo, c.co + lo, c.vlo + lo, c.vuo + lo};
    for (int k = 0; k < EpiKktColDist::NIN; ++k) cd.in[k] = in[k];
    epilogue_walk<EpiKktColDist><<<c.grid_nside, kBlock, 0, s>>>(c.nside, cd, c.partAt);
    k_sum_partials<6><<<1, kBlock, 0, s>>>(c.partAt, c.grid_nside, c.ksum + 4);
    CK(cudaGetLastError());
    allreduce(c, c.ksum, 10, s);
    k_kkt_from_sums<<<1, 32, 0, s>>>(c.ctl, c.ksum);
    CK(cudaGetLastError());
  } else {
    // local rows; the last block publishes the row-side sums into xchg[n+8..n+12)
    EpiKktRowDist rd{};
    static_cast<EpiKktRow&>(rd) = er;
    rd.xsums = c.xchg + c.n + 8;
    launch_spmv(c, c.A, c.grid_a, xs, rd, c.partA, &c.ctl->ticket_kkt, c.stream);
    launch_spmv(c, c.At, c.grid_at, ys, store_into(c.xchg), nullptr, nullptr, c.stream);
    allreduce(c, c.xchg, static_cast<size_t>(c.n) + 16, c.stream);
    EpiKktColDist cd{};
    cd.col = ec;
    const double* in[] = {c.xchg, xs, c.cs, c.co, c.vlo, c.vuo};
    for (int k = 0; k < EpiKktColDist::NIN; ++k) cd.in[k] = in[k];
    epilogue_walk<EpiKktColDist><<<nside_grid(c), kBlock, 0, c.stream>>>(nside_sched(c), cd, c.partAt);
    CK(cudaGetLastError());
    k_kkt_dist_finalize<<<1, kBlock, 0, c.stream>>>(c.ctl, c.partAt, nside_grid(c),
                                                    nside_sched(c).n_multi, nside_long_red(c),
                                                    c.xchg + c.n + 8);
    CK(cudaGetLastError());
  }
  pull_ctl(c);
  const Ctl& h = *c.ctl_host;
  out->primal_value = h.kkt_cx;
  out->py = h.kkt_py;
  out->pr = h.kkt_pr;
  out->viol2 = h.kkt_viol2;
  out->eq2 = h.kkt_eq2;
  out->cone2 = h.kkt_cone2;
  out->py_inf = static_cast<int64_t>(h.kkt_py_inf);
  out->pr_inf = static_cast<int64_t>(h.kkt_pr_inf);
  out->nan_x = static_cast<int64_t>(h.kkt_nan_x);
  out->nan_y = static_cast<int64_t>(h.kkt_nan_y);
}

void exact_caches(rhp_ctx& c) {
  // z.ax = A x, z.aty = A^T y
  launch_spmv(c, c.A, c.grid_a, c.x, store_into(c.ax), nullptr, nullptr, c.stream);
  launch_spmv(c, c.At, c.grid_at, c.y, store_into(c.aty), nullptr, nullptr, c.stream);
}

}  // namespace

extern "C" {

const char* rhp_last_error(void) { return g_err.c_str(); }
}  // extern "C"

// ops.cu reports its failures through the same thread-local message
void rhp_internal_set_error(const std::string& msg) { g_err = msg; }

extern "C" {

int rhp_device_count(int* count) {
  return guarded([&] {
    *count = 0;
    const cudaError_t e = cudaGetDeviceCount(count);
    if (e != cudaSuccess) {
      cudaGetLastError();
      *count = 0;
    }
  });
}

int rhp_get_device_info(int device, rhp_device_info* info) {
  return guarded([&] {
    cudaDeviceProp p{};
    CK(cudaGetDeviceProperties(&p, device));
    std::memset(info, 0, sizeof(*info));
    std::snprintf(info->name, sizeof(info->name), "%s", p.name);
    info->sm_count = p.multiProcessorCount;
    info->cc_major = p.major;
    info->cc_minor = p.minor;
    info->l2_bytes = p.l2CacheSize;
    info->mem_bytes = static_cast<int64_t>(p.totalGlobalMem);
    int rt = 0;
    CK(cudaRuntimeGetVersion(&rt));
    info->graph_supported = rt >= 12040 ? 1 : 0;
  });
}

int rhp_local_group_create(int world, void** out) {
  return guarded([&] {
    if (world < 1) throw std::invalid_argument("rhp_local_group_create: world must be >= 1");
    *out = new LocalGroup(world);
  });
}

int rhp_local_group_destroy(void* group) {
  delete static_cast<LocalGroup*>(group);
  return RHPDHG_OK;
}

int rhp_nccl_unique_id(void* out128) {
  return guarded([&] {
#ifdef RHP_WITH_NCCL
    ncclUniqueId id;
    if (nccl().GetUniqueId(&id) != ncclSuccess) throw CudaError("ncclGetUniqueId failed");
    std::memcpy(out128, &id, sizeof(id));
#else
    (void)out128;
    throw CudaError("built without NCCL");
#endif
  });
}

int rhp_create(const rhpdhg_lp_view* lp, const rhp_options* opt_in, rhp_ctx** out) {
  *out = nullptr;
  rhp_ctx* c = new rhp_ctx();
  // RHPDHG_SETUP_TRACE=1: per-phase times of the context build on stderr
  const bool trace = std::getenv("RHPDHG_SETUP_TRACE") != nullptr;
  auto tp = std::chrono::steady_clock::now();
  auto phase = [&](const char* what) {
    if (!trace) return;
    cudaDeviceSynchronize();
    const auto now = std::chrono::steady_clock::now();
    std::fprintf(stderr, "  create %-22s %9.3f s\n", what, std::chrono::duration<double>(now - tp).count());
    tp = now;
  };
  const int rc = guarded([&] {
    rhp_options opt{};
    opt.device = 0;
    opt.rank = 0;
    opt.world_size = 1;
    opt.use_graph = 1;
    opt.block_limit = 64;
    opt.resident = -1;
    if (opt_in) opt = *opt_in;
    if (opt.block_limit < 1) opt.block_limit = 64;
    if (opt.world_size < 1 || opt.rank < 0 || opt.rank >= opt.world_size)
      throw std::invalid_argument("rhp_create: bad rank/world_size");
    if (opt.world_size > 1 && !opt.nccl_id && !opt.local_group)
      throw std::invalid_argument("rhp_create: world_size > 1 needs an NCCL unique id or a local group");
    if (opt.nccl_id && opt.local_group)
      throw std::invalid_argument("rhp_create: give an NCCL id or a local group, not both");
    if (opt.local_group && static_cast<const LocalGroup*>(opt.local_group)->world != opt.world_size)
      throw std::invalid_argument("rhp_create: local group size differs from world_size");
    // row-partitioned path (also with one rank when an id is given: parity tests)
    c->dist = opt.nccl_id != nullptr || opt.local_group != nullptr;
    c->rank = opt.rank;
    c->world = opt.world_size;
    {
      const char* pe = std::getenv("RHP_PEER_EXCHANGE");
      const char* rep = std::getenv("RHP_DIST_REPLICATED");
      c->sharded = c->dist && c->world > 1 && !(pe && pe[0] == '1') && !(rep && rep[0] == '1');
    }
    if (c->dist) opt.use_graph = 0;  // NCCL calls are launched from the host loop
    c->opt = opt;
    if (lp->num_cons < 0 || lp->num_vars < 0 || lp->nnz < 0)
      throw std::invalid_argument("matrix dimensions must be nonnegative");
    CK(cudaSetDevice(opt.device));
    cudaDeviceProp p{};
    CK(cudaGetDeviceProperties(&p, opt.device));
    if (p.major < 10)
      throw CudaError("rhpdhg device library is built for sm_100a (B200); device is sm_" +
                      std::to_string(p.major) + std::to_string(p.minor));
    c->sm_count = p.multiProcessorCount;
    CK(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
    CK(cudaEventCreate(&c->ev0));
    CK(cudaEventCreate(&c->ev1));
    CK(cudaEventCreate(&c->tev0));
    CK(cudaEventCreate(&c->tev1));
    if (c->dist) {
      c->offsets = partition_rows(*lp, c->world);
      for (int r = 0; r < c->world; ++r)
        c->max_local = std::max(c->max_local, c->offsets[r + 1] - c->offsets[r]);
      ingest_device(*lp, c->offsets[c->rank], c->offsets[c->rank + 1], c->L, c->A, c->At, -1, c->stream);
    } else {
      phase("device init");
      int locality = opt.locality;
      if (const char* e = std::getenv("RHP_LOCALITY")) locality = std::atoi(e);
      ingest_device(*lp, 0, lp->num_cons, c->L, c->A, c->At, locality, c->stream);
    }
    phase("ingest");
    const HostLayout& L = c->L;
    c->m = L.m;
    c->n = L.n;
    cudaStream_t s = c->stream;
    const size_t m = static_cast<size_t>(c->m), n = static_cast<size_t>(c->n);
    c->nalloc = c->n;
    if (c->sharded) {
      c->S = (c->n + c->world - 1) / c->world;
      c->nlo = std::min<int64_t>(c->n, c->S * c->rank);
      c->nhi = std::min<int64_t>(c->n, c->nlo + c->S);
      c->nalloc = std::max<int64_t>(c->n, c->S * c->world);  // in-place all-gathers
    }
    for (double** p2 : {&c->c, &c->vl, &c->vu, &c->co, &c->vlo, &c->vuo, &c->cs, &c->x, &c->aty,
                        &c->x0, &c->aty0, &c->xp, &c->xout, &c->rcout, &c->pv, &c->pw})
      *p2 = dev_alloc<double>(static_cast<size_t>(c->nalloc));
    for (double** p2 : {&c->cl, &c->cu, &c->clo, &c->cuo, &c->rs, &c->y, &c->ax, &c->y0, &c->ax0,
                        &c->yp, &c->yout, &c->pav})
      *p2 = dev_alloc<double>(m);
    const std::vector<int32_t> lrows = local_rows(*c);
    upload_perm(c->co, lp->objective, L.pcol, c->hbuf, s);
    upload_perm(c->vlo, lp->var_lb, L.pcol, c->hbuf, s);
    upload_perm(c->vuo, lp->var_ub, L.pcol, c->hbuf, s);
    upload_perm(c->clo, lp->con_lb, L.prow, c->hbuf, s);
    upload_perm(c->cuo, lp->con_ub, L.prow, c->hbuf, s);
    CK(cudaMemcpyAsync(c->c, c->co, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(c->vl, c->vlo, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(c->vu, c->vuo, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(c->cl, c->clo, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
    CK(cudaMemcpyAsync(c->cu, c->cuo, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
    c->hbuf.assign(std::max(m, n), 1.0);
    upload(c->rs, c->hbuf.data(), m, s);
    upload(c->cs, c->hbuf.data(), n, s);
    CK(cudaStreamSynchronize(s));
    // grids: persistent, a multiple of the SM count, never more than tiles
    // one grid per operator: every kernel walking it must see the same CTA count
    const int occ_store = prepare_spmv<EpiStore>();
    int occ_a = std::min({prepare_spmv<EpiDual>(), prepare_spmv<EpiKktRow>(),
                          prepare_spmv<EpiKktRowDist>(), occ_store});
    if (!c->dist && kRowsMinBlocks > kMinBlocks && thread_rows_rule(c->L.A.rp))
      occ_a = std::min({prepare_rows<EpiDual>(), prepare_rows<EpiKktRow>(), prepare_rows<EpiStore>()});
    int occ_at = std::min({prepare_spmv<EpiAty>(), prepare_spmv<EpiKktCol>(),
                           prepare_spmv<EpiPowerW>(), occ_store});
    // A^T walked by the thread-per-row engine only (single GPU: its walkers
    // are spmv_rows and K3's epilogue_walk, grid-stride loops over the same
    // thread map): the grid follows the rows kernel's own register budget
    // (RHP_ROWS_MIN_BLOCKS)
    if (!c->dist && kRowsMinBlocks > kMinBlocks && thread_rows_rule(c->L.At.rp))
      occ_at = std::min({prepare_rows<EpiAty>(), prepare_rows<EpiKktCol>(), prepare_rows<EpiPowerW>(),
                         prepare_rows<EpiStore>()});
    // at least ~2 windows of work per warp, at most every resident CTA
    auto clampg = [](const HostOperator& h, int64_t cap) {
      const int64_t work = h.nnz + 2 * h.rows;
      return static_cast<int>(std::max<int64_t>(1, std::min(cap, work / (2 * kWin * kWarps))));
    };
    c->grid_a = clampg(c->L.A, (int64_t)c->sm_count * occ_a);
    c->grid_at = clampg(c->L.At, (int64_t)c->sm_count * occ_at);
    build_schedule(c->L.A, (int64_t)c->grid_a * kWarps, kRowWeight);
    build_schedule(c->L.At, (int64_t)c->grid_at * kWarps, kRowWeight);
    phase("vectors");
    upload_sched(c->A, c->L.A, s);
    upload_sched(c->At, c->L.At, s);
    phase("schedules");
    c->grid_vec = vec_grid(*c, std::max<int64_t>(c->m, c->n));
    // rank-independent n-side map (partitioned path): n and the device are
    // the same on every rank, so is this grid
    // sharded: the walk covers the owned slice; S (not the slice length) sets
    // the grid, so it is the same on every rank
    c->grid_nside = vec_grid(*c, c->sharded ? c->S : c->n);
    c->nside.thread_rows = 1;
    c->nside.rows = c->sharded ? c->nhi - c->nlo : c->n;
    c->grid_max = std::max({c->grid_a, c->grid_at, c->grid_vec, c->grid_nside});
    for (double** p2 : {&c->part1, &c->part3, &c->partA, &c->partAt})
      *p2 = dev_alloc<double>(static_cast<size_t>(c->grid_max) * 16);
    c->hist = dev_alloc<double>(static_cast<size_t>(opt.block_limit));
    if (const char* e = std::getenv("RHP_PDL")) c->pdl = e[0] == '1';
    choose_engines(*c);
    choose_gather_policy(*c);
    phase("engines+gather tuning");
    CK(cudaMalloc(&c->ctl, sizeof(Ctl)));
    CK(cudaMallocHost(&c->ctl_host, sizeof(Ctl)));
    std::memset(c->ctl_host, 0, sizeof(Ctl));
    Ctl& h = *c->ctl_host;
    h.graph_mode = opt.use_graph ? 1 : 0;
    h.hist = c->hist;
    h.block_limit = opt.block_limit;
    h.check_interval = 64;
    h.iteration_limit = INT64_MAX;
    h.r_anchor = h.r_prev = std::numeric_limits<double>::infinity();
    h.k1_token = -1;
    CK(cudaMemcpy(c->ctl, c->ctl_host, sizeof(Ctl), cudaMemcpyHostToDevice));
    for (double* p2 : {c->x, c->aty, c->x0, c->aty0, c->xp, c->xout, c->rcout, c->pv, c->pw})
      CK(cudaMemsetAsync(p2, 0, std::max<size_t>(n, 1) * sizeof(double), s));
    for (double* p2 : {c->y, c->ax, c->y0, c->ax0, c->yp, c->yout, c->pav})
      CK(cudaMemsetAsync(p2, 0, std::max<size_t>(m, 1) * sizeof(double), s));
    c->xchg = dev_alloc<double>(static_cast<size_t>(c->nalloc) + 16);  // zero tail: RS padding
    if (c->sharded) {
      c->rsb = dev_alloc<double>(static_cast<size_t>(c->S) + 8);
      c->dsum = dev_alloc<double>(16);
      c->ksum = dev_alloc<double>(16);
    }
    CK(cudaStreamSynchronize(s));
    // small LPs: one cluster runs whole blocks when its CSR slices fit in
    // shared memory (auto) or when forced
    c->resident = !c->dist && opt.resident != 0 && setup_resident(*c);
    phase("resident check");
    if (c->dist) {
      c->ypad = dev_alloc<double>(static_cast<size_t>(c->max_local));
      c->ygather = dev_alloc<double>(static_cast<size_t>(c->max_local) * c->world);
      c->agree = dev_alloc<int64_t>(1);
      if (opt.local_group) {
        c->comm = std::make_unique<LocalComm>(
            static_cast<LocalGroup*>(const_cast<void*>(opt.local_group)), c->rank);
      } else {
#ifdef RHP_WITH_NCCL
        c->comm = std::make_unique<NcclComm>(opt.nccl_id, c->world, c->rank);
#else
        throw CudaError("built without NCCL");
#endif
      }
      if (const char* e = std::getenv("RHP_PEER_EXCHANGE"); e && e[0] == '1') setup_peers(*c);
      CK(cudaHostAlloc(&c->stop_mirror, sizeof(int) * static_cast<size_t>(opt.block_limit),
                       cudaHostAllocMapped));
      CK(cudaHostGetDevicePointer(reinterpret_cast<void**>(&c->stop_mirror_dev), c->stop_mirror, 0));
      c->it_events.resize(static_cast<size_t>(opt.block_limit));
      for (cudaEvent_t& e : c->it_events) CK(cudaEventCreateWithFlags(&e, cudaEventDisableTiming));
      SET_CTL(*c, stop_mirror, c->stop_mirror_dev);
    }
  });
  if (rc != RHPDHG_OK) {
    rhp_destroy(c);
    return rc;
  }
  *out = c;
  return RHPDHG_OK;
}

int rhp_destroy(rhp_ctx* c) {
  if (!c) return RHPDHG_OK;
  if (c->stream) cudaStreamSynchronize(c->stream);
  if (c->gexec) cudaGraphExecDestroy(c->gexec);
  if (c->graph) cudaGraphDestroy(c->graph);
  for (void* p : c->peer_opened) cudaIpcCloseMemHandle(p);
  if (c->peer_ticket) cudaFree(c->peer_ticket);
  free_op(c->A);
  free_op(c->At);
  for (double* p : {c->c, c->vl, c->vu, c->cl, c->cu, c->co, c->vlo, c->vuo, c->clo, c->cuo,
                    c->rs, c->cs, c->x, c->y, c->ax, c->aty, c->x0, c->y0, c->ax0, c->aty0,
                    c->xp, c->yp, c->xout, c->yout, c->rcout, c->pv, c->pw, c->pav, c->part1,
                    c->part3, c->partA, c->partAt, c->hist, c->xchg, c->ypad, c->ygather})
    if (p) cudaFree(p);
  if (c->agree) cudaFree(c->agree);
  if (c->opbuf) cudaFree(c->opbuf);
  for (double* p : {c->rsb, c->dsum, c->ksum})
    if (p) cudaFree(p);
  if (c->csc_src) cudaFree(c->csc_src);
  if (c->res_a_split) cudaFree(c->res_a_split);
  if (c->res_at_split) cudaFree(c->res_at_split);
  c->comm.reset();
  if (c->stop_mirror) cudaFreeHost(c->stop_mirror);
  for (cudaEvent_t e : c->it_events) cudaEventDestroy(e);
  if (c->ctl) cudaFree(c->ctl);
  if (c->ctl_host) cudaFreeHost(c->ctl_host);
  if (c->ev0) cudaEventDestroy(c->ev0);
  if (c->ev1) cudaEventDestroy(c->ev1);
  if (c->tev0) cudaEventDestroy(c->tev0);
  if (c->tev1) cudaEventDestroy(c->tev1);
  if (c->stream) cudaStreamDestroy(c->stream);
  delete c;
  return RHPDHG_OK;
}

int rhp_layout(rhp_ctx* c, rhp_layout_info* info) {
  return guarded([&] {
    std::memset(info, 0, sizeof(*info));
    info->m_local = c->m;
    info->n = c->n;
    info->nnz_local = c->L.nnz;
    for (int k = 0; k < 8; ++k) {
      info->row_bins[k] = c->L.A.bin_rows[k];
      info->col_bins[k] = c->L.At.bin_rows[k];
    }
    info->grid_a = c->grid_a;
    info->grid_at = c->grid_at;
    info->grid_vec = c->grid_vec;
    info->sm_count = c->sm_count;
    info->gather_l1 = (c->A.l1g ? 1 : 0) | (c->At.l1g ? 2 : 0);
    info->pdl = c->pdl ? 1 : 0;
    info->thread_rows = (fin(c->A).sched.thread_rows ? 1 : 0) | (fin(c->At).sched.thread_rows ? 2 : 0) |
                        (c->A.cta_row ? 4 : 0) | (fin(c->A).sell_ci ? 8 : 0) |
                        (fin(c->At).sell_ci ? 16 : 0) | (fin(c->A).sched.uniform_len ? 32 : 0) |
                        (fin(c->At).sched.uniform_len ? 64 : 0) | (c->A.row_band ? 128 : 0) |
                        (c->At.row_band ? 256 : 0);
    info->resident = c->resident ? 1 : 0;
    info->partition = !c->dist ? 0 : c->sharded ? 2 : 1;
    info->const_bounds = static_cast<int32_t>(c->const_mask);
    info->relabel = c->L.relabel ? 1 : 0;
    for (int k = 0; k < 4; ++k) info->sectors[k] = c->L.sectors[k];
    info->segments = static_cast<int32_t>(std::max<size_t>(1, c->A.segs.size()) |
                                          (std::max<size_t>(1, c->At.segs.size()) << 16));
  });
}

// ruiz_equilibrate + pock_chambolle_scale (scaling.cpp:46-81) on the device.
int rhp_scale(rhp_ctx* c, int enabled, int ruiz_iterations, int pock_chambolle) {
  return guarded([&] {
    // the original values are consumed (freed below) and rs/cs accumulate:
    // scaling twice would compound the scales from already-scaled values
    if (c->scaled) throw std::invalid_argument("rhp_scale: the context is already scaled");
    c->scaled = true;
    cudaStream_t s = c->stream;
    const int64_t m = c->m, n = c->n;
    const int gr = vec_grid(*c, std::max<int64_t>(m, n));
    if (enabled) {
      // Ruiz on working copies of the original values (A.v and At.v hold
      // the originals until the final apply)
      double* rmax = c->pav;  // m scratch
      double* cmax = c->pw;   // n scratch
      double* wA = c->A.v;
      double* wT = c->At.v;
      for (int pass = 0; pass < ruiz_iterations; ++pass) {
        k_row_absmax_sqrt<<<gr, kBlock, 0, s>>>(c->A.rp, wA, m, rmax);
        if (!c->dist) {
          k_row_absmax_sqrt<<<gr, kBlock, 0, s>>>(c->At.rp, wT, n, cmax);
        } else {  // column maxima over all ranks' rows (max is exact: order-free)
          k_row_absmax_raw<<<gr, kBlock, 0, s>>>(c->At.rp, wT, n, cmax);
          allreduce_max(*c, cmax, static_cast<size_t>(n), s);
          k_sqrt_or_one<<<gr, kBlock, 0, s>>>(cmax, n);
        }
        k_ruiz_divide<<<gr, kBlock, 0, s>>>(c->A.rp, c->A.ci, wA, m, rmax, cmax);
        k_ruiz_divide<<<gr, kBlock, 0, s>>>(c->At.rp, c->At.ci, wT, n, cmax, rmax);
        k_vec_div<<<gr, kBlock, 0, s>>>(c->rs, rmax, m);
        k_vec_div<<<gr, kBlock, 0, s>>>(c->cs, cmax, n);
      }
      // apply_scales(original, rs, cs): values and vectors from the originals
      k_scale_values<<<gr, kBlock, 0, s>>>(c->A.rp, c->A.ci, c->A.v_orig, c->A.v, m, c->rs, c->cs);
      k_scale_values<<<gr, kBlock, 0, s>>>(c->At.rp, c->At.ci,
                                           c->csc_src ? c->csc_src : c->At.v_orig, c->At.v, n, c->cs,
                                           c->rs);
      k_apply_col_scales<<<gr, kBlock, 0, s>>>(c->c, c->vl, c->vu, c->cs, n);
      k_apply_row_scales<<<gr, kBlock, 0, s>>>(c->cl, c->cu, c->rs, m);
      if (pock_chambolle) {
        double* rn = c->pav;
        double* cn = c->pw;
        k_pc_rows<<<gr, kBlock, 0, s>>>(c->A.rp, c->A.v, m, rn);
        if (!c->dist) {
          k_pc_cols<<<gr, kBlock, 0, s>>>(c->At.rp, c->At.ci, c->At.v_orig, n, c->rs, c->cs, cn);
        } else {  // per-rank partial 1-norms, summed across ranks
          k_pc_cols_raw<<<gr, kBlock, 0, s>>>(c->At.rp, c->At.ci, c->At.v_orig, n, c->rs, c->cs,
                                              cn);
          allreduce(*c, cn, static_cast<size_t>(n), s);
          k_inv_sqrt_or_one<<<gr, kBlock, 0, s>>>(cn, n);
        }
        // apply_scales(ruiz-scaled, rn, cn) in place
        k_scale_values<<<gr, kBlock, 0, s>>>(c->A.rp, c->A.ci, c->A.v, c->A.v, m, rn, cn);
        k_scale_values<<<gr, kBlock, 0, s>>>(c->At.rp, c->At.ci, c->At.v, c->At.v, n, cn, rn);
        k_apply_col_scales<<<gr, kBlock, 0, s>>>(c->c, c->vl, c->vu, cn, n);
        k_apply_row_scales<<<gr, kBlock, 0, s>>>(c->cl, c->cu, rn, m);
        k_vec_mul<<<gr, kBlock, 0, s>>>(c->rs, rn, m);
        k_vec_mul<<<gr, kBlock, 0, s>>>(c->cs, cn, n);
      }
      CK(cudaGetLastError());
    }
    // the original values are no longer needed on the device
    CK(cudaStreamSynchronize(s));
    if (c->A.v_orig) CK(cudaFree(c->A.v_orig));
    if (c->At.v_orig) CK(cudaFree(c->At.v_orig));
    c->A.v_orig = c->At.v_orig = nullptr;
    if (c->csc_src) CK(cudaFree(c->csc_src));
    c->csc_src = nullptr;
    detect_constant_inputs(*c);
    // column segments of the scaled operators (gathered vectors larger than L2)
    build_segments(*c, c->A, c->L.A, c->n, c->grid_a);
    build_segments(*c, c->At, c->L.At, c->m, c->grid_at);
    carve_row_band(*c, c->A, c->n, c->grid_a);
    carve_row_band(*c, c->At, c->m, c->grid_at);
    build_sliced(*c, c->A);
    build_sliced(*c, c->At);
    if (c->graph_built) {  // the block graph captured the unsegmented launches
      CK(cudaGraphExecDestroy(c->gexec));
      CK(cudaGraphDestroy(c->graph));
      c->gexec = nullptr;
      c->graph = nullptr;
      c->graph_built = false;
    }
  });
}

int rhp_get_scaled(rhp_ctx* c, const rhp_scaled_out* o) {
  return guarded([&] {
    const HostLayout& L = c->L;
    const std::vector<int32_t> lrows = local_rows(*c);
    // device element order = the reference's CSR / CSC order (not on a
    // relabelled layout: the matrix values are only available unrelabelled)
    const size_t nz = static_cast<size_t>(L.nnz);
    if ((o->csr_values || o->csc_values) && nz && c->L.relabel)
      throw std::invalid_argument("rhp_get_scaled: matrix values of a relabelled layout");
    if (o->csr_values && nz) CK(cudaMemcpy(o->csr_values, c->A.v, nz * sizeof(double), cudaMemcpyDeviceToHost));
    if (o->csc_values && nz) CK(cudaMemcpy(o->csc_values, c->At.v, nz * sizeof(double), cudaMemcpyDeviceToHost));
    if (o->row_scale) download_perm(o->row_scale, c->rs, lrows, c->hbuf, c->stream);
    if (o->col_scale) download_perm(o->col_scale, c->cs, L.pcol, c->hbuf, c->stream);
    if (o->objective) download_perm(o->objective, c->c, L.pcol, c->hbuf, c->stream);
    if (o->var_lb) download_perm(o->var_lb, c->vl, L.pcol, c->hbuf, c->stream);
    if (o->var_ub) download_perm(o->var_ub, c->vu, L.pcol, c->hbuf, c->stream);
    if (o->con_lb) download_perm(o->con_lb, c->cl, lrows, c->hbuf, c->stream);
    if (o->con_ub) download_perm(o->con_ub, c->cu, lrows, c->hbuf, c->stream);
  });
}

int rhp_power_begin(rhp_ctx* c, const double* v0) {
  return guarded([&] { upload_perm(c->pv, v0, c->L.pcol, c->hbuf, c->stream); });
}

int rhp_power_step(rhp_ctx* c, double* vw, double* ww) {
  return guarded([&] {
    launch_spmv(*c, c->A, c->grid_a, c->pv, store_into(c->pav), nullptr, nullptr, c->stream);
    if (!c->dist) {
      EpiPowerW e{};
      e.ctl = c->ctl;
      e.w = c->pw;
      e.in[0] = c->pv;
      launch_spmv(*c, c->At, c->grid_at, c->pav, e, c->partAt, &c->ctl->ticket_pow, c->stream);
    } else if (c->sharded) {  // owned slice of w = sum_p A_p^T (A_p v); dots allreduced
      const int64_t lo = c->nlo;
      launch_spmv(*c, c->At, c->grid_at, c->pav, store_into(c->xchg), nullptr, nullptr, c->stream);
      c->comm->reduce_scatter(c->xchg, c->rsb, static_cast<size_t>(c->S), c->stream);
      EpiPowerDist e{};
      e.w = c->pw + lo;
      e.in[0] = c->rsb;
      e.in[1] = c->pv + lo;
      epilogue_walk<EpiPowerDist><<<c->grid_nside, kBlock, 0, c->stream>>>(c->nside, e, c->partAt);
      k_sum_partials<2><<<1, kBlock, 0, c->stream>>>(c->partAt, c->grid_nside, c->ksum);
      CK(cudaGetLastError());
      allreduce(*c, c->ksum, 2, c->stream);
      k_power_from_sums<<<1, 32, 0, c->stream>>>(c->ctl, c->ksum);
      CK(cudaGetLastError());
    } else {  // w = sum over ranks of A_p^T (A_p v), then v.w and w.w redundantly
      launch_spmv(*c, c->At, c->grid_at, c->pav, store_into(c->xchg), nullptr, nullptr,
                  c->stream);
      allreduce(*c, c->xchg, static_cast<size_t>(c->n), c->stream);
      EpiPowerDist e{};
      e.w = c->pw;
      e.in[0] = c->xchg;
      e.in[1] = c->pv;
      epilogue_walk<EpiPowerDist><<<nside_grid(*c), kBlock, 0, c->stream>>>(nside_sched(*c), e, c->partAt);
      k_power_dist_finalize<<<1, kBlock, 0, c->stream>>>(c->ctl, c->partAt, nside_grid(*c),
                                                         nside_sched(*c).n_multi, nside_long_red(*c));
      CK(cudaGetLastError());
    }
    pull_ctl(*c);
    *vw = c->ctl_host->pw_vw;
    *ww = c->ctl_host->pw_ww;
  });
}

int rhp_power_normalize(rhp_ctx* c, double wnorm) {
  return guarded([&] {
    k_normalize<<<c->grid_vec, kBlock, 0, c->stream>>>(c->pv, c->pw, wnorm, c->n);
    CK(cudaGetLastError());
    // sharded: only the owned slice of w is current; every rank's slice of v
    if (c->sharded)
      c->comm->allgather(c->pv + c->S * c->rank, c->pv, static_cast<size_t>(c->S) * sizeof(double),
                         c->stream);
  });
}

int rhp_spmv(rhp_ctx* c, int transpose, const double* in, double* out) {
  return guarded([&] {
    const std::vector<int32_t> lrows = local_rows(*c);
    if (!transpose) {
      upload_perm(c->pv, in, c->L.pcol, c->hbuf, c->stream);
      launch_spmv(*c, c->A, c->grid_a, c->pv, store_into(c->pav), nullptr, nullptr, c->stream);
      download_perm(out, c->pav, lrows, c->hbuf, c->stream);
    } else {
      upload_perm(c->pav, in, lrows, c->hbuf, c->stream);
      launch_spmv(*c, c->At, c->grid_at, c->pav, store_into(c->pw), nullptr, nullptr, c->stream);
      download_perm(out, c->pw, c->L.pcol, c->hbuf, c->stream);
    }
  });
}

int rhp_set_step(rhp_ctx* c, const rhp_step* st) {
  return guarded([&] {
    pull_ctl(*c);
    Ctl& h = *c->ctl_host;
    h.eta = st->eta;
    h.omega = st->omega;
    h.gamma = st->gamma;
    h.tau = st->tau;
    h.sigma = st->sigma;
    h.sigma_inv = st->sigma_inv;
    h.primal_scale = st->primal_scale;
    h.dual_scale = st->dual_scale;
    h.beta_s = st->beta_sufficient;
    h.beta_n = st->beta_necessary;
    h.beta_a = st->beta_artificial;
    h.check_interval = st->check_interval;
    h.iteration_limit = st->iteration_limit;
    h.restarts_enabled = st->restarts_enabled;
    h.record_history = st->record_history;
    c->host_check_interval = st->check_interval;
    c->host_iteration_limit = st->iteration_limit;
    CK(cudaMemcpyAsync(c->ctl, c->ctl_host, offsetof(Ctl, k), cudaMemcpyHostToDevice, c->stream));
    CK(cudaStreamSynchronize(c->stream));
  });
}

int rhp_reset_iterate(rhp_ctx* c) {
  return guarded([&] {
    cudaStream_t s = c->stream;
    const size_t m = static_cast<size_t>(std::max<int64_t>(c->m, 1));
    const size_t n = static_cast<size_t>(std::max<int64_t>(c->n, 1));
    for (double* p : {c->x, c->aty, c->x0, c->aty0, c->xp})
      CK(cudaMemsetAsync(p, 0, n * sizeof(double), s));
    for (double* p : {c->y, c->ax, c->y0, c->ax0, c->yp})
      CK(cudaMemsetAsync(p, 0, m * sizeof(double), s));
    pull_ctl(*c);
    Ctl& h = *c->ctl_host;
    h.k = 0;
    h.total = 0;
    h.block_iters = 0;
    h.r_anchor = h.r_prev = std::numeric_limits<double>::infinity();
    h.r_last = 0.0;
    h.stop = h.verdict = h.check_due = h.breakdown = 0;
    h.k1_token = -1;
    h.x_dist2 = h.y_dist2 = h.x_norm2 = h.y_norm2 = 0.0;
    CK(cudaMemcpyAsync(c->ctl, c->ctl_host, sizeof(Ctl), cudaMemcpyHostToDevice, s));
    CK(cudaStreamSynchronize(s));
    c->host_total = 0;
  });
}

int rhp_set_iterate(rhp_ctx* c, const double* x, const double* y) {
  return guarded([&] {
    upload_perm(c->x, x, c->L.pcol, c->hbuf, c->stream);
    upload_perm(c->y, y, local_rows(*c), c->hbuf, c->stream);
    exact_caches(*c);
    CK(cudaStreamSynchronize(c->stream));
  });
}

int rhp_run_block(rhp_ctx* c, rhp_block_out* out) {
  return guarded([&] {
    cudaStream_t s = c->stream;
    CK(cudaEventRecord(c->ev0, s));
    if (c->resident) {
      launch_resident(*c, s);
    } else if (c->opt.use_graph) {
      if (!c->graph_built) build_graph(*c);
      CK(cudaGraphLaunch(c->gexec, s));
    } else {
      // plain launches: enough iterations to reach the next stop point;
      // kernels of iterations past the stop exit at entry
      int64_t L = c->opt.block_limit;
      const int64_t ci = c->host_check_interval;
      L = std::min<int64_t>(L, ci - (c->host_total % ci));
      if (c->host_iteration_limit != INT64_MAX)
        L = std::min<int64_t>(L, std::max<int64_t>(1, c->host_iteration_limit - c->host_total));
      launch_primal_init(*c, s);
      if (!c->dist) {
        for (int64_t i = 0; i < L; ++i) launch_iteration(*c, static_cast<int>(i), s);
      } else {
        // partitioned: iteration i's control kernel writes its stop flag to
        // mapped host memory; the host launches at most kPollAhead iterations
        // past the last flag it has seen, so after an on-device stop (restart
        // verdict mid-block) at most kPollAhead no-op iterations, and their
        // collectives, are issued — instead of the rest of the block
        constexpr int64_t kPollAhead = 2;
        std::fill(c->stop_mirror, c->stop_mirror + L, 0);
        for (int64_t i = 0; i < L; ++i) {
          if (i >= kPollAhead) {
            CK(cudaEventSynchronize(c->it_events[i - kPollAhead]));
            if (reinterpret_cast<volatile int*>(c->stop_mirror)[i - kPollAhead]) break;
          }
          launch_iteration(*c, static_cast<int>(i), s);
          CK(cudaEventRecord(c->it_events[i], s));
        }
      }
    }
    CK(cudaEventRecord(c->ev1, s));
    pull_ctl(*c);
    float ms = 0.f;
    CK(cudaEventElapsedTime(&ms, c->ev0, c->ev1));
    c->last_block_ms = ms;
    const Ctl& h = *c->ctl_host;
    c->host_total = h.total;
    out->iterations_done = h.block_iters;
    out->total = h.total;
    out->k = h.k;
    out->verdict = h.verdict;
    out->check_due = h.check_due;
    out->breakdown = h.breakdown;
    out->r_last = h.r_last;
    out->r_anchor = h.r_anchor;
    out->r_prev = h.r_prev;
    out->q_last = h.q_last;
    out->x_dist2 = h.x_dist2;
    out->y_dist2 = h.y_dist2;
    out->x_norm2 = h.x_norm2;
    out->y_norm2 = h.y_norm2;
  });
}

int rhp_get_history(rhp_ctx* c, double* out, int64_t cap, int64_t* count) {
  return guarded([&] {
    const int64_t k = std::min<int64_t>(c->ctl_host->block_iters, cap);
    if (k > 0) CK(cudaMemcpy(out, c->hist, static_cast<size_t>(k) * sizeof(double),
                             cudaMemcpyDeviceToHost));
    *count = k;
  });
}

int rhp_kkt(rhp_ctx* c, int which, rhp_kkt_sums* out) {
  return guarded([&] {
    if (which == 0) run_kkt(*c, c->x, c->y, true, true, out);
    else run_kkt(*c, c->xp, c->yp, false, false, out);
  });
}

int rhp_kkt_of(rhp_ctx* c, const double* x, const double* y, rhp_kkt_sums* out) {
  return guarded([&] {
    // scratch: pv (n) and pav (m); the scales are still 1 before rhp_scale
    upload_perm(c->pv, x, c->L.pcol, c->hbuf, c->stream);
    upload_perm(c->pav, y, local_rows(*c), c->hbuf, c->stream);
    run_kkt(*c, c->pv, c->pav, false, false, out);
  });
}

// Row-partitioned: every rank receives the full m-vector (rank blocks are
// contiguous original rows; NCCL allgather of the padded local blocks).
void gather_rows(rhp_ctx& c, const double* dev_local, double* host_full) {
  cudaStream_t s = c.stream;
  const size_t ml = static_cast<size_t>(c.m), mx = static_cast<size_t>(c.max_local);
  CK(cudaMemsetAsync(c.ypad, 0, std::max<size_t>(mx, 1) * sizeof(double), s));
  if (ml) CK(cudaMemcpyAsync(c.ypad, dev_local, ml * sizeof(double), cudaMemcpyDeviceToDevice, s));
  c.comm->allgather(c.ypad, c.ygather, mx * sizeof(double), s);
  std::vector<double> all(mx * static_cast<size_t>(c.world));
  if (!all.empty())
    CK(cudaMemcpyAsync(all.data(), c.ygather, all.size() * sizeof(double), cudaMemcpyDeviceToHost,
                       s));
  CK(cudaStreamSynchronize(s));
  for (int r = 0; r < c.world; ++r)
    std::copy(all.begin() + static_cast<ptrdiff_t>(r * mx),
              all.begin() + static_cast<ptrdiff_t>(r * mx + (c.offsets[r + 1] - c.offsets[r])),
              host_full + c.offsets[r]);
}

int rhp_fetch_solution(rhp_ctx* c, double* x, double* y, double* rcost) {
  return guarded([&] {
    if (c->sharded) {  // the owners' slices of the unscaled x and reduced costs
      const size_t b = static_cast<size_t>(c->S) * sizeof(double);
      c->comm->allgather(c->xout + c->S * c->rank, c->xout, b, c->stream);
      c->comm->allgather(c->rcout + c->S * c->rank, c->rcout, b, c->stream);
    }
    if (x) download_perm(x, c->xout, c->L.pcol, c->hbuf, c->stream);
    if (y) {
      if (c->dist) gather_rows(*c, c->yout, y);
      else download_perm(y, c->yout, local_rows(*c), c->hbuf, c->stream);
    }
    if (rcost) download_perm(rcost, c->rcout, c->L.pcol, c->hbuf, c->stream);
  });
}

int rhp_partition_rows(const rhpdhg_lp_view* lp, int world_size, int64_t* offsets) {
  return guarded([&] {
    if (world_size < 1) throw std::invalid_argument("world_size must be >= 1");
    const std::vector<int64_t> off = partition_rows(*lp, world_size);
    std::copy(off.begin(), off.end(), offsets);
  });
}

int rhp_any(rhp_ctx* c, int flag, int* any) {
  return guarded([&] {
    if (!c->dist) {
      *any = flag;
      return;
    }
    int64_t v = flag ? 1 : 0;
    CK(cudaMemcpyAsync(c->agree, &v, sizeof v, cudaMemcpyHostToDevice, c->stream));
    c->comm->allreduce_max_i64(c->agree, 1, c->stream);
    CK(cudaMemcpyAsync(&v, c->agree, sizeof v, cudaMemcpyDeviceToHost, c->stream));
    CK(cudaStreamSynchronize(c->stream));
    *any = v != 0;
  });
}

int rhp_fetch_iterate(rhp_ctx* c, double* x, double* y, double* ax, double* aty) {
  return guarded([&] {
    if (c->sharded) {
      const size_t b = static_cast<size_t>(c->S) * sizeof(double);
      c->comm->allgather(c->x + c->S * c->rank, c->x, b, c->stream);
      c->comm->allgather(c->aty + c->S * c->rank, c->aty, b, c->stream);
    }
    const std::vector<int32_t> lrows = local_rows(*c);
    if (x) download_perm(x, c->x, c->L.pcol, c->hbuf, c->stream);
    if (y) download_perm(y, c->y, lrows, c->hbuf, c->stream);
    if (ax) download_perm(ax, c->ax, lrows, c->hbuf, c->stream);
    if (aty) download_perm(aty, c->aty, c->L.pcol, c->hbuf, c->stream);
  });
}

int rhp_restart(rhp_ctx* c) {
  return guarded([&] {
    cudaStream_t s = c->stream;
    const size_t m = static_cast<size_t>(c->m), n = static_cast<size_t>(c->n);
    if (n) {
      CK(cudaMemcpyAsync(c->x0, c->x, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(c->aty0, c->aty, n * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    if (m) {
      CK(cudaMemcpyAsync(c->y0, c->y, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
      CK(cudaMemcpyAsync(c->ax0, c->ax, m * sizeof(double), cudaMemcpyDeviceToDevice, s));
    }
    const double inf = std::numeric_limits<double>::infinity();
    const int64_t zero = 0;
    SET_CTL(*c, k, zero);
    SET_CTL(*c, r_anchor, inf);
    SET_CTL(*c, r_prev, inf);
  });
}

int rhp_last_block_ms(rhp_ctx* c, double* ms) {
  *ms = c->last_block_ms;
  return RHPDHG_OK;
}

int rhp_timer(rhp_ctx* c, int start, double* ms) {
  return guarded([&] {
    if (start) {
      CK(cudaEventRecord(c->tev0, c->stream));
      if (ms) *ms = 0.0;
    } else {
      CK(cudaEventRecord(c->tev1, c->stream));
      CK(cudaEventSynchronize(c->tev1));
      float f = 0.f;
      CK(cudaEventElapsedTime(&f, c->tev0, c->tev1));
      if (ms) *ms = f;
    }
  });
}

// Times `reps` back-to-back launches of each fused iteration kernel on the
// live iterate (CUDA events on the ctx stream). Mutates the iterate: call
// after the measured solve work is done.
int rhp_time_kernels(rhp_ctx* c, int reps, double* ms_k1, double* ms_k2, double* ms_k3) {
  return guarded([&] {
    cudaStream_t s = c->stream;
    pull_ctl(*c);
    const int32_t gm = c->ctl_host->graph_mode;
    const int32_t zero = 0, one = 1;
    SET_CTL(*c, graph_mode, zero);
    SET_CTL(*c, bench, one);
    float f = 0.f;
    CK(cudaEventRecord(c->tev0, s));
    for (int r = 0; r < reps; ++r) launch_primal_init(*c, s);
    CK(cudaEventRecord(c->tev1, s));
    CK(cudaEventSynchronize(c->tev1));
    CK(cudaEventElapsedTime(&f, c->tev0, c->tev1));
    if (ms_k3) *ms_k3 = f / reps;
    CK(cudaEventRecord(c->tev0, s));
    for (int r = 0; r < reps; ++r)
      launch_spmv(*c, c->A, c->grid_a, c->xp, epi_dual(*c, 0), c->part1, &c->ctl->ticket_dual, s);
    CK(cudaEventRecord(c->tev1, s));
    CK(cudaEventSynchronize(c->tev1));
    CK(cudaEventElapsedTime(&f, c->tev0, c->tev1));
    if (ms_k1) *ms_k1 = f / reps;
    CK(cudaEventRecord(c->tev0, s));
    for (int r = 0; r < reps; ++r)
      launch_spmv(*c, c->At, c->grid_at, c->yp, epi_aty(*c, 0), c->part3, nullptr, s);
    CK(cudaEventRecord(c->tev1, s));
    CK(cudaEventSynchronize(c->tev1));
    CK(cudaEventElapsedTime(&f, c->tev0, c->tev1));
    if (ms_k2) *ms_k2 = f / reps;
    SET_CTL(*c, bench, zero);
    SET_CTL(*c, graph_mode, gm);
  });
}

// Average device ms of `reps` plain SpMVs (out = A v or A^T v, no epilogue
// reductions) on the current matrix: the SpMV engine's own rate.
int rhp_gather_ceiling(rhp_ctx* c, int reps, double* ms_a, double* ms_at) {
  return guarded([&] {
    cudaStream_t s = c->stream;
    int occ = 0;
    CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(
        &occ, reinterpret_cast<const void*>(k_gather_probe<false>), 256, 0));
    const int grid = c->sm_count * std::max(occ, 1);
    double* out = nullptr;
    CK(cudaMalloc(&out, static_cast<size_t>(grid) * 256 * sizeof(double)));
    auto run1 = [&](const DevOp& op, const double* x) {
      if (op.l1g) k_gather_probe<true><<<grid, 256, 0, s>>>(op.ci, op.v, x, op.nnz, out);
      else k_gather_probe<false><<<grid, 256, 0, s>>>(op.ci, op.v, x, op.nnz, out);
    };
    auto run = [&](const DevOp& op, const double* x) {  // segment by segment when segmented
      if (op.segs.empty()) run1(op, x);
      for (const DevOp& g : op.segs) run1(g, x);
    };
    for (auto [op, x, ms] : {std::tuple<const DevOp*, const double*, double*>{&c->A, c->xp, ms_a},
                             {&c->At, c->yp, ms_at}}) {
      if (!ms) continue;
      run(*op, x);  // warm-up
      float best = 1e30f;
      for (int r = 0; r < std::max(reps, 1); ++r) {
        CK(cudaEventRecord(c->tev0, s));
        run(*op, x);
        CK(cudaEventRecord(c->tev1, s));
        CK(cudaEventSynchronize(c->tev1));
        float f = 0.f;
        CK(cudaEventElapsedTime(&f, c->tev0, c->tev1));
        best = std::min(best, f);
      }
      *ms = best;
    }
    CK(cudaGetLastError());
    CK(cudaFree(out));
  });
}

int rhp_time_spmv(rhp_ctx* c, int transpose, int reps, double* ms) {
  return guarded([&] {
    cudaStream_t s = c->stream;
    float f = 0.f;
    CK(cudaEventRecord(c->tev0, s));
    for (int r = 0; r < reps; ++r) {
      if (transpose)
        launch_spmv(*c, c->At, c->grid_at, c->pav, store_into(c->pw), nullptr, nullptr, s);
      else
        launch_spmv(*c, c->A, c->grid_a, c->pv, store_into(c->pav), nullptr, nullptr, s);
    }
    CK(cudaEventRecord(c->tev1, s));
    CK(cudaEventSynchronize(c->tev1));
    CK(cudaEventElapsedTime(&f, c->tev0, c->tev1));
    *ms = f / reps;
  });
}

int rhp_profiler_range(int start) {
  return guarded([&] { CK(start ? cudaProfilerStart() : cudaProfilerStop()); });
}

int rhp_synchronize(rhp_ctx* c) {
  return guarded([&] { CK(cudaStreamSynchronize(c->stream)); });
}

// ---------------------------------------------------------------- per-op --
// The reference's per-operation API as device round trips (rhpdhg_cuda.h).

int rhp_set_vectors(rhp_ctx* c, const rhp_op_lp* lp) {
  return guarded([&] {
    if (c->scaled || c->dist)
      throw std::invalid_argument("rhp_set_vectors: needs an unscaled single-GPU context");
    cudaStream_t s = c->stream;
    const std::vector<int32_t> lrows = local_rows(*c);
    upload_perm(c->co, lp->objective, c->L.pcol, c->hbuf, s);
    upload_perm(c->vlo, lp->var_lb, c->L.pcol, c->hbuf, s);
    upload_perm(c->vuo, lp->var_ub, c->L.pcol, c->hbuf, s);
    upload_perm(c->clo, lp->con_lb, lrows, c->hbuf, s);
    upload_perm(c->cuo, lp->con_ub, lrows, c->hbuf, s);
  });
}

int rhp_set_csc_values(rhp_ctx* c, const double* csc_values, int scale_source) {
  return guarded([&] {
    if (c->scaled || c->dist || c->L.relabel)
      throw std::invalid_argument("rhp_set_csc_values: needs an unscaled, unrelabelled single-GPU context");
    const size_t nz = static_cast<size_t>(c->L.nnz);
    if (!nz) return;
    if (scale_source) {
      if (!c->csc_src) c->csc_src = dev_alloc<double>(nz);
      upload(c->csc_src, csc_values, nz, c->stream);
    } else {
      upload(c->At.v, csc_values, nz, c->stream);
    }
    CK(cudaStreamSynchronize(c->stream));
  });
}

int rhp_op_pdhg(rhp_ctx* c, const rhp_op_params* p, const rhp_op_lp* lp, const rhp_op_iter* z,
                const rhp_op_iter* anchor, const rhp_op_out* inner, double* dx, double* dy,
                const rhp_op_out* znew) {
  return guarded([&] {
    if (c->scaled || c->dist)
      throw std::invalid_argument("rhp_op_pdhg: needs an unscaled single-GPU context");
    cudaStream_t s = c->stream;
    const int64_t m = c->m, n = c->n;
    const size_t mp = static_cast<size_t>(std::max<int64_t>(m, 1)) + 8;
    const size_t np = static_cast<size_t>(std::max<int64_t>(n, 1)) + 8;
    if (!c->opbuf) c->opbuf = dev_alloc<double>(12 * np + 11 * mp);
    double* b = c->opbuf;
    double *x = b, *aty = b + np, *cc = b + 2 * np, *lb = b + 3 * np, *ub = b + 4 * np,
           *xp = b + 5 * np, *atyp = b + 6 * np, *ddx = b + 7 * np, *x0 = b + 8 * np,
           *aty0 = b + 9 * np, *xn = b + 10 * np, *atyn = b + 11 * np;
    double* bm = b + 12 * np;
    double *y = bm, *ax = bm + mp, *cl = bm + 2 * mp, *cu = bm + 3 * mp, *yp = bm + 4 * mp,
           *axp = bm + 5 * mp, *ddy = bm + 6 * mp, *y0 = bm + 7 * mp, *ax0 = bm + 8 * mp,
           *yn = bm + 9 * mp, *axn = bm + 10 * mp;
    const std::vector<int32_t> lrows = local_rows(*c);
    upload_perm(x, z->x, c->L.pcol, c->hbuf, s);
    upload_perm(aty, z->aty, c->L.pcol, c->hbuf, s);
    upload_perm(y, z->y, lrows, c->hbuf, s);
    upload_perm(ax, z->ax, lrows, c->hbuf, s);
    upload_perm(cc, lp->objective, c->L.pcol, c->hbuf, s);
    upload_perm(lb, lp->var_lb, c->L.pcol, c->hbuf, s);
    upload_perm(ub, lp->var_ub, c->L.pcol, c->hbuf, s);
    upload_perm(cl, lp->con_lb, lrows, c->hbuf, s);
    upload_perm(cu, lp->con_ub, lrows, c->hbuf, s);
    const int gn = vec_grid(*c, n), gm = vec_grid(*c, m);
    // x+ = proj(x - tau(c - aty)); ax+ = A x+
    k_op_primal<<<gn, kBlock, 0, s>>>(n, p->tau, x, aty, cc, lb, ub, xp);
    CK(cudaGetLastError());
    if (c->L.nnz > 0 && m > 0) launch_spmv(*c, c->A, c->grid_a, xp, store_into(axp), nullptr, nullptr, s);
    else if (m > 0) CK(cudaMemsetAsync(axp, 0, static_cast<size_t>(m) * sizeof(double), s));
    // y+ from the caches (2 ax+ - ax); aty+ = A^T y+
    k_op_dual<<<gm, kBlock, 0, s>>>(m, p->sigma, p->sigma_inv, y, ax, axp, cl, cu, yp);
    CK(cudaGetLastError());
    if (c->L.nnz > 0 && n > 0) launch_spmv(*c, c->At, c->grid_at, yp, store_into(atyp), nullptr, nullptr, s);
    else if (n > 0) CK(cudaMemsetAsync(atyp, 0, static_cast<size_t>(n) * sizeof(double), s));
    k_op_sub<<<gn, kBlock, 0, s>>>(n, x, xp, ddx);
    k_op_sub<<<gm, kBlock, 0, s>>>(m, y, yp, ddy);
    CK(cudaGetLastError());
    if (anchor && znew) {
      upload_perm(x0, anchor->x, c->L.pcol, c->hbuf, s);
      upload_perm(aty0, anchor->aty, c->L.pcol, c->hbuf, s);
      upload_perm(y0, anchor->y, lrows, c->hbuf, s);
      upload_perm(ax0, anchor->ax, lrows, c->hbuf, s);
      k_op_affine<<<gn, kBlock, 0, s>>>(n, p->a, p->gamma, p->b, xp, x, x0, xn);
      k_op_affine<<<gm, kBlock, 0, s>>>(m, p->a, p->gamma, p->b, yp, y, y0, yn);
      k_op_affine<<<gm, kBlock, 0, s>>>(m, p->a, p->gamma, p->b, axp, ax, ax0, axn);
      k_op_affine<<<gn, kBlock, 0, s>>>(n, p->a, p->gamma, p->b, atyp, aty, aty0, atyn);
      CK(cudaGetLastError());
      download_perm(znew->x, xn, c->L.pcol, c->hbuf, s);
      download_perm(znew->y, yn, lrows, c->hbuf, s);
      download_perm(znew->ax, axn, lrows, c->hbuf, s);
      download_perm(znew->aty, atyn, c->L.pcol, c->hbuf, s);
    }
    download_perm(inner->x, xp, c->L.pcol, c->hbuf, s);
    download_perm(inner->y, yp, lrows, c->hbuf, s);
    download_perm(inner->ax, axp, lrows, c->hbuf, s);
    download_perm(inner->aty, atyp, c->L.pcol, c->hbuf, s);
    if (dx) download_perm(dx, ddx, c->L.pcol, c->hbuf, s);
    if (dy) download_perm(dy, ddy, lrows, c->hbuf, s);
  });
}

}  // extern "C"
