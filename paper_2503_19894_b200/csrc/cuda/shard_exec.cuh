// Sharded execution (include/tilesim/shard.hpp schedules) -- included at the
// end of runtime.cu, whose handle types and launch helpers it shares.
//
//  tsg_vshard_run  2^g virtual shards on one device; a swap is one in-place
//                  kernel over each shard pair (single-GPU emulation of the
//                  distributed path, used by the GPU parity tests)
//  tsg_dist_*      one process per GPU of a box.  Shards are exported with
//                  CUDA IPC, so every rank addresses every peer's shard
//                  directly (NVLink / NVSwitch peer memory).  A Swap op is
//                  ONE in-place kernel per slab (k_exchange): the bit
//                  transpositions G_i <-> L_i of the op form an involution
//                  of the global index; each element pair is swapped by
//                  exactly one rank (a peer load + a peer store, no staging,
//                  no pack / unpack), all pairs of the op at once (a grouped
//                  all-to-all).  Exchanges run on a comm stream; the only
//                  host synchronisation is a shared-memory barrier that
//                  orders interprocess-event records before peers' waits.
//                  Pipelined swaps (ShardOp::pipeline_bits) overlap the
//                  exchange of slab c with the local gates on slab c - 1.
#include <unistd.h>

#include "../host/rendezvous.hpp"

namespace {

// ------------------------------------------------------------------ kernels
__device__ __forceinline__ uint64_t with_bit(uint64_t i, int b, uint64_t v) {
  const uint64_t low = i & ((uint64_t{1} << b) - 1);
  return ((i >> b) << (b + 1)) | (v << b) | low;
}

// shard `a` (rank bit 0) gives its bit-b = 1 half, shard `c` (rank bit 1) its
// bit-b = 0 half; element i of the half index space pairs the two
template <typename Real>
__global__ void k_swap_halves(Real* __restrict__ a, Real* __restrict__ c, uint64_t half, int b) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < half; i += stride) {
    const uint64_t la = with_bit(i, b, 1), lc = la ^ (uint64_t{1} << b);
    const Real t = a[la];
    a[la] = c[lc];
    c[lc] = t;
  }
}

// In-place exchange of one Swap op over peer memory.  Physical index
// P = (rank << nl) | l.  sigma swaps bit (nl + gbit[i]) with bit lpos[i] for
// every pair i -- an involution.  An element with L-bits v (its lpos bits)
// differing from the rank's G-bits u moves to rank r' (G-bits <- v) at local
// l' (L-bits <- u).  The pair {(r, l), (r', l')} is swapped by exactly one
// side: the one whose `zbit` (a local bit sigma leaves alone) equals
// (r < r') ? 0 : 1 -- both sides see the same zbit, and opposite orders.
// A launch covers one slab (T bits = slab); T and zbit are never L bits.
constexpr int kMaxRanks = 64;
constexpr int kMaxPipelineBits = 3;
template <typename Real, int V>
struct ExVec;
template <> struct ExVec<double, 1> { using T = double; };
template <> struct ExVec<double, 2> { using T = double2; };
template <> struct ExVec<float, 1> { using T = float; };
template <> struct ExVec<float, 4> { using T = float4; };
struct ExchangeParams {
  void* re[kMaxRanks];
  void* im[kMaxRanks];
  int nl, rank, m, zbit, tlo;
  int gbit[6], lpos[6];
  uint64_t slab;    // value of the T bits [tlo, nl)
  uint64_t n_work;  // work items (V consecutive elements each) per launch
};

template <typename Real, int V>
__global__ void __launch_bounds__(512) k_exchange(const __grid_constant__ ExchangeParams p) {
  using Vec = typename ExVec<Real, V>::T;
  uint32_t u = 0;
  for (int i = 0; i < p.m; ++i) u |= ((static_cast<uint32_t>(p.rank) >> p.gbit[i]) & 1u) << i;
  Real* my_re = static_cast<Real*>(p.re[p.rank]);
  Real* my_im = static_cast<Real*>(p.im[p.rank]);
  const uint64_t zlow = (uint64_t{1} << p.zbit) - 1;
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t w = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; w < p.n_work; w += stride) {
    const uint64_t x = w * V;  // bits of l other than T and zbit
    uint64_t l = ((x & ~zlow) << 1) | (x & zlow) | (p.slab << p.tlo);
    uint32_t v = 0;
    for (int i = 0; i < p.m; ++i) v |= static_cast<uint32_t>((l >> p.lpos[i]) & 1u) << i;
    if (v == u) continue;  // stays on this rank
    int peer = p.rank;
    uint64_t lp = l;
    for (int i = 0; i < p.m; ++i) {
      peer = (peer & ~(1 << p.gbit[i])) | static_cast<int>(((v >> i) & 1u) << p.gbit[i]);
      lp = (lp & ~(uint64_t{1} << p.lpos[i])) | (static_cast<uint64_t>((u >> i) & 1u) << p.lpos[i]);
    }
    const uint64_t zv = p.rank < peer ? 0 : 1;  // this side owns the pairs with zbit == zv
    l |= zv << p.zbit;
    lp |= zv << p.zbit;
    Real* pr = static_cast<Real*>(p.re[peer]);
    Real* pi = static_cast<Real*>(p.im[peer]);
    const Vec a_re = *reinterpret_cast<const Vec*>(my_re + l);
    const Vec a_im = *reinterpret_cast<const Vec*>(my_im + l);
    const Vec b_re = *reinterpret_cast<const Vec*>(pr + lp);
    const Vec b_im = *reinterpret_cast<const Vec*>(pi + lp);
    *reinterpret_cast<Vec*>(my_re + l) = b_re;
    *reinterpret_cast<Vec*>(my_im + l) = b_im;
    *reinterpret_cast<Vec*>(pr + lp) = a_re;
    *reinterpret_cast<Vec*>(pi + lp) = a_im;
  }
}

// exchange parameters of a Swap op on a rank (peer pointers filled at run time)
ExchangeParams exchange_params(const ShardOp& op, int nl, int rank, int pipeline_bits) {
  ExchangeParams p;
  std::memset(&p, 0, sizeof p);
  p.nl = nl;
  p.rank = rank;
  p.m = static_cast<int>(op.swaps.size());
  if (p.m > 6) throw SimError("exchange of more than 6 qubit pairs");
  uint64_t lmask = 0;
  for (int i = 0; i < p.m; ++i) {
    p.gbit[i] = op.swaps[i].first - nl;
    p.lpos[i] = op.swaps[i].second;
    lmask |= uint64_t{1} << p.lpos[i];
  }
  p.tlo = nl - pipeline_bits;
  // owner bit: the highest local position below T that no pair moves
  p.zbit = -1;
  for (int b = p.tlo - 1; b >= 0 && p.zbit < 0; --b)
    if (!((lmask >> b) & 1u)) p.zbit = b;
  if (p.zbit < 0) throw SimError("exchange needs a local qubit outside the swapped ones");
  return p;
}

// ------------------------------------------------------- prepared schedule
// A rank's share of a ShardPlan: segments of consecutive local work (each
// one program: tile passes, block splits, diagonal batches, as on one GPU)
// and the exchanges between them.
struct DistItem {
  bool swap = false;
  // segment
  tsg_program* full = nullptr;  // over the whole shard
  tsg_program* slab = nullptr;  // over one slab (n_local - pipeline_bits qubits) when the preceding swap pipelines
  uint64_t launches = 0;
  // swap
  ExchangeParams xp{};
  int pipeline_bits = 0;
  uint64_t moved_bytes = 0;  // bytes this rank sends (one direction)
};

struct PreparedRank {
  std::vector<DistItem> items;
  ~PreparedRank() {
    for (DistItem& it : items) {
      if (it.full) tsg_program_destroy(it.full);
      if (it.slab) tsg_program_destroy(it.slab);
    }
  }
};

std::unique_ptr<PreparedRank> prepare_rank(const ShardPlan& plan, uint64_t rank, int prec, tsg_ctx* ctx) {
  auto pr = std::make_unique<PreparedRank>();
  const int nl = plan.n_local;
  const uint64_t amp = prec == 64 ? 16 : 8;
  Circuit seg;  // the open run of local gates (this rank's sub-gates)
  seg.n_qubits = nl;
  int slab_bits = 0;    // pipeline bits of the swap that opened the segment
  int prefix_left = 0;  // ops of the pipelined prefix still to come
  auto close_segment = [&]() {
    if (seg.gates.empty()) return;
    DistItem it;
    it.full = build_program(ctx, seg, plan.zero_tol, plan.one_tol, prec).release();
    it.launches = it.full->launches;
    if (slab_bits > 0) {
      Circuit sc = seg;
      sc.n_qubits = nl - slab_bits;
      it.slab = build_program(ctx, sc, plan.zero_tol, plan.one_tol, prec).release();
      it.launches = it.slab->launches << slab_bits;
    }
    pr->items.push_back(std::move(it));
    seg.gates.clear();
  };
  for (const ShardOp& op : plan.ops) {
    if (op.kind == ShardOp::Kind::Swap) {
      close_segment();
      DistItem it;
      it.swap = true;
      it.pipeline_bits = op.pipeline_bits;
      it.xp = exchange_params(op, nl, static_cast<int>(rank), op.pipeline_bits);
      it.moved_bytes = (uint64_t{1} << nl) / (uint64_t{1} << it.xp.m) * ((uint64_t{1} << it.xp.m) - 1) * amp;
      pr->items.push_back(std::move(it));
      slab_bits = op.pipeline_ops > 0 ? op.pipeline_bits : 0;
      prefix_left = slab_bits > 0 ? op.pipeline_ops : 0;
      continue;
    }
    // the pipelined prefix is its own segment (slab programs); the rest of
    // the run of local ops starts a plain one
    auto count_prefix = [&]() {
      if (prefix_left > 0 && --prefix_left == 0) {
        close_segment();
        slab_bits = 0;
      }
    };
    Gate g = op.kind == ShardOp::Kind::Local ? op.gate : rank_subgate(op, nl, rank);
    if (g.k() == 0) {  // every target global: a rank-wide phase, as diag(v, v) on local qubit 0
      const cplx v = g.matrix.at(0, 0);
      if (v == cplx(1.0, 0.0)) {
        count_prefix();
        continue;
      }
      GateMatrix m(1);
      m.at(0, 0) = v;
      m.at(1, 1) = v;
      g = make_gate(std::move(m), {0});
    }
    seg.gates.push_back(std::move(g));
    count_prefix();
  }
  close_segment();
  return pr;
}

template <typename Real>
void launch_exchange(const ExchangeParams& base, int pipeline_bits, uint64_t slab, cudaStream_t s, int max_ctas) {
  ExchangeParams p = base;
  p.slab = slab;
  // V consecutive elements per item when no swapped bit, owner bit or slab
  // bit sits below log2 V (16-byte accesses)
  constexpr int VMAX = sizeof(Real) == 8 ? 2 : 4;
  int low = p.zbit;
  for (int i = 0; i < p.m; ++i) low = std::min(low, p.lpos[i]);
  const uint64_t items = uint64_t{1} << (p.nl - pipeline_bits - 1);
  const unsigned threads = 512;
  auto grid = [&](uint64_t work) {
    return static_cast<unsigned>(std::max<uint64_t>(1, std::min<uint64_t>((work + threads - 1) / threads, max_ctas)));
  };
  if ((1 << low) >= VMAX && items >= static_cast<uint64_t>(VMAX)) {
    p.n_work = items / VMAX;
    k_exchange<Real, VMAX><<<grid(p.n_work), threads, 0, s>>>(p);
  } else {
    p.n_work = items;
    k_exchange<Real, 1><<<grid(p.n_work), threads, 0, s>>>(p);
  }
  ck(cudaGetLastError(), "k_exchange");
}

uint64_t run_segment(const DistItem& it, tsg_state* st) {
  run_program(st, it.full, nullptr);
  return it.full->launches;
}

}  // namespace

struct tsg_dist {
  tsg_ctx* ctx = nullptr;
  tsg_state* st = nullptr;  // this rank's 2^n_local shard
  int n = 0, n_global = 0, rank = 0, world = 1;
  std::unique_ptr<tilesim::ShmRendezvous> rv;
  void* peer_re[kMaxRanks] = {};
  void* peer_im[kMaxRanks] = {};
  cudaStream_t comm = nullptr;
  // interprocess events (own, and peers' opened from their handles)
  cudaEvent_t ready = nullptr, done[1 << kMaxPipelineBits] = {};
  cudaEvent_t peer_ready[kMaxRanks] = {}, peer_done[kMaxRanks][1 << kMaxPipelineBits] = {};
  // timing
  cudaEvent_t e0 = nullptr, e1 = nullptr;
  std::vector<cudaEvent_t> xt;  // pairs around exchanges, grown on demand
  int exchange_ctas = 64;
  // prepared schedules keyed by the plan's serial (never reused, unlike its address)
  std::map<uint64_t, std::unique_ptr<PreparedRank>> prepared;
  std::vector<uint64_t> prepared_order;
};

namespace {

struct DistSlot {  // one rank's rendezvous payload
  cudaIpcMemHandle_t re, im;
  cudaIpcEventHandle_t ready, done[1 << kMaxPipelineBits];
  int device;
  int pid;
};

const PreparedRank& prepared_for(tsg_dist* d, const tsc_shard_plan* plan) {
  auto it = d->prepared.find(plan->serial);
  if (it != d->prepared.end()) return *it->second;
  if (d->prepared.size() >= 16) {  // bound the cache: drop the oldest schedule
    d->prepared.erase(d->prepared_order.front());
    d->prepared_order.erase(d->prepared_order.begin());
  }
  d->prepared_order.push_back(plan->serial);
  return *d->prepared.emplace(plan->serial, prepare_rank(plan->plan, d->rank, d->st->prec, d->ctx)).first->second;
}

cudaEvent_t xt_event(tsg_dist* d, size_t i) {
  while (d->xt.size() <= i) {
    cudaEvent_t e;
    ck(cudaEventCreate(&e), "event");
    d->xt.push_back(e);
  }
  return d->xt[i];
}

// One Swap item (and, when it pipelines, the segment after it).  Returns
// the kernels launched; `*consumed` tells the caller the next segment ran.
uint64_t dist_exchange(tsg_dist* d, const DistItem& sw, const DistItem* next, size_t xi, bool* consumed) {
  cudaStream_t s = d->st->stream;
  const int C = 1 << sw.pipeline_bits;
  ExchangeParams xp = sw.xp;
  for (int r = 0; r < d->world; ++r) {
    xp.re[r] = d->peer_re[r];
    xp.im[r] = d->peer_im[r];
  }
  // every rank's earlier work on its shard is done before anyone touches it
  ck(cudaEventRecord(d->ready, s), "record ready");
  d->rv->barrier();  // all ready records issued
  ck(cudaStreamWaitEvent(d->comm, d->ready, 0), "wait ready");
  for (int r = 0; r < d->world; ++r)
    if (r != d->rank) ck(cudaStreamWaitEvent(d->comm, d->peer_ready[r], 0), "wait peer ready");
  ck(cudaEventRecord(xt_event(d, 2 * xi), d->comm), "event");
  for (int c = 0; c < C; ++c) {
    if (d->st->prec == 64) launch_exchange<double>(xp, sw.pipeline_bits, c, d->comm, d->exchange_ctas);
    else launch_exchange<float>(xp, sw.pipeline_bits, c, d->comm, d->exchange_ctas);
    ck(cudaEventRecord(d->done[c], d->comm), "record done");
  }
  ck(cudaEventRecord(xt_event(d, 2 * xi + 1), d->comm), "event");
  d->rv->barrier();  // all done records issued
  uint64_t launches = C;
  *consumed = false;
  if (sw.pipeline_bits > 0 && next && !next->swap && next->slab) {
    // slab c of every shard is final once every rank finished its batch c
    const int nlocal = d->st->n - sw.pipeline_bits;
    for (int c = 0; c < C; ++c) {
      ck(cudaStreamWaitEvent(s, d->done[c], 0), "wait done");
      for (int r = 0; r < d->world; ++r)
        if (r != d->rank) ck(cudaStreamWaitEvent(s, d->peer_done[r][c], 0), "wait peer done");
      tsg_state view = *d->st;
      view.n = nlocal;
      const size_t off = (static_cast<size_t>(c) << nlocal) * d->st->amp_bytes();
      view.re = static_cast<unsigned char*>(d->st->re) + off;
      view.im = static_cast<unsigned char*>(d->st->im) + off;
      run_program(&view, next->slab, nullptr);
      launches += next->slab->launches;
    }
    *consumed = true;
  } else {
    ck(cudaStreamWaitEvent(s, d->done[C - 1], 0), "wait done");
    for (int r = 0; r < d->world; ++r)
      if (r != d->rank) ck(cudaStreamWaitEvent(s, d->peer_done[r][C - 1], 0), "wait peer done");
  }
  return launches;
}

}  // namespace

extern "C" {

int tsg_vshard_run(tsg_ctx* ctx, const tsc_shard_plan* plan, int precision_bits, const double* re_in,
                   const double* im_in, double* re_out, double* im_out, tsg_run_report* report) {
  TSG_TRY({
    require(ctx && plan && re_in && im_in && re_out && im_out, "null argument");
    require(precision_bits == 64 || precision_bits == 32, "precision_bits must be 64 or 32");
    const ShardPlan& sp = plan->plan;
    const int nl = sp.n_local, g = sp.n_global;
    require(nl >= 1 && g <= 6, "virtual sharding supports up to 64 shards");
    use_device(ctx);
    const uint64_t S = uint64_t{1} << g, local = uint64_t{1} << nl;
    std::vector<std::unique_ptr<tsg_state, int (*)(tsg_state*)>> shards;
    std::vector<std::unique_ptr<PreparedRank>> prep;
    for (uint64_t s = 0; s < S; ++s) {
      tsg_state* st = nullptr;
      if (tsg_state_create(ctx, nl, precision_bits, &st)) throw SimError(tsg_last_error());
      shards.emplace_back(st, tsg_state_destroy);
      if (tsg_state_upload(st, re_in + s * local, im_in + s * local)) throw SimError(tsg_last_error());
      prep.push_back(prepare_rank(sp, s, precision_bits, ctx));
    }
    // one stream orders every shard's launches and the exchanges (the
    // shards' own streams are restored before they are destroyed)
    cudaStream_t stream = shards[0]->stream;
    std::vector<cudaStream_t> own(S);
    for (uint64_t s = 0; s < S; ++s) {
      own[s] = shards[s]->stream;
      shards[s]->stream = stream;
    }
    struct Restore {
      std::vector<std::unique_ptr<tsg_state, int (*)(tsg_state*)>>& sh;
      std::vector<cudaStream_t>& own;
      ~Restore() {
        for (size_t s = 0; s < sh.size(); ++s) sh[s]->stream = own[s];
      }
    } restore{shards, own};
    cudaEvent_t e0, e1;
    ck(cudaEventCreate(&e0), "event");
    ck(cudaEventCreate(&e1), "event");
    ck(cudaEventRecord(e0, stream), "event");
    uint64_t exchanged = 0, launches = 0;
    const size_t n_items = prep[0]->items.size();
    for (size_t i = 0; i < n_items; ++i) {
      if (prep[0]->items[i].swap) {
        // every virtual rank runs its share of the pairs (k_exchange, the
        // distributed kernel itself), slab by slab
        const DistItem& sw0 = prep[0]->items[i];
        for (int c = 0; c < (1 << sw0.pipeline_bits); ++c)
          for (uint64_t s = 0; s < S; ++s) {
            ExchangeParams xp = prep[s]->items[i].xp;
            for (uint64_t r = 0; r < S; ++r) {
              xp.re[r] = shards[r]->re;
              xp.im[r] = shards[r]->im;
            }
            if (precision_bits == 64) launch_exchange<double>(xp, sw0.pipeline_bits, c, stream, 1024);
            else launch_exchange<float>(xp, sw0.pipeline_bits, c, stream, 1024);
            ++launches;
          }
        exchanged += sw0.moved_bytes;
        continue;
      }
      for (uint64_t s = 0; s < S; ++s) {
        require(i < prep[s]->items.size() && !prep[s]->items[i].swap, "ranks disagree on the schedule");
        launches += run_segment(prep[s]->items[i], shards[s].get());
      }
    }
    ck(cudaEventRecord(e1, stream), "event");
    ck(cudaEventSynchronize(e1), "vshard sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, e0, e1), "elapsed");
    cudaEventDestroy(e0);
    cudaEventDestroy(e1);
    // gather: physical index (s << nl) | l, then undo the qubit map
    std::vector<double> pre(S * local), pim(S * local);
    for (uint64_t s = 0; s < S; ++s)
      if (tsg_state_download(shards[s].get(), pre.data() + s * local, pim.data() + s * local))
        throw SimError(tsg_last_error());
    for (uint64_t x = 0; x < S * local; ++x) {
      const uint64_t p = physical_index(x, sp.final_pos);
      re_out[x] = pre[p];
      im_out[x] = pim[p];
    }
    if (report) {
      *report = tsg_run_report{};
      report->execution_s = ms * 1e-3;
      report->gates = sp.ops.size();
      report->launches = launches;
      report->exchanged_bytes = exchanged;
    }
  })
}

int tsg_dist_unique_id(unsigned char id[128]) {
  TSG_TRY({
    require(id != nullptr, "null argument");
    tilesim::ShmRendezvous::make_id(id);
  })
}

int tsg_dist_create(tsg_ctx* ctx, int n_qubits, int precision_bits, int n_global, int rank, const unsigned char id[128],
                    tsg_dist** out) {
  TSG_TRY({
    require(ctx && id && out, "null argument");
    require(n_global >= 0 && n_global <= 6 && n_global < n_qubits, "n_global must be in [0, min(n, 7))");
    require(rank >= 0 && rank < (1 << n_global), "rank out of range");
    use_device(ctx);
    auto d = std::make_unique<tsg_dist>();
    d->ctx = ctx;
    d->n = n_qubits;
    d->n_global = n_global;
    d->rank = rank;
    d->world = 1 << n_global;
    if (const char* e = std::getenv("TSG_EXCHANGE_CTAS")) d->exchange_ctas = std::max(1, std::atoi(e));
    if (tsg_state_create(ctx, n_qubits - n_global, precision_bits, &d->st)) throw SimError(tsg_last_error());
    ck(cudaStreamCreateWithFlags(&d->comm, cudaStreamNonBlocking), "comm stream");
    ck(cudaEventCreate(&d->e0), "event");
    ck(cudaEventCreate(&d->e1), "event");
    const unsigned ipc_flags = cudaEventDisableTiming | (d->world > 1 ? cudaEventInterprocess : 0);
    ck(cudaEventCreateWithFlags(&d->ready, ipc_flags), "event");
    for (cudaEvent_t& e : d->done) ck(cudaEventCreateWithFlags(&e, ipc_flags), "event");
    d->peer_re[rank] = d->st->re;
    d->peer_im[rank] = d->st->im;
    d->rv = std::make_unique<tilesim::ShmRendezvous>(id, rank, d->world, sizeof(DistSlot));
    if (d->world > 1) {
      DistSlot* mine = static_cast<DistSlot*>(d->rv->slot(rank));
      ck(cudaIpcGetMemHandle(&mine->re, d->st->re), "ipc handle re");
      ck(cudaIpcGetMemHandle(&mine->im, d->st->im), "ipc handle im");
      ck(cudaIpcGetEventHandle(&mine->ready, d->ready), "ipc event");
      for (int c = 0; c < (1 << kMaxPipelineBits); ++c) ck(cudaIpcGetEventHandle(&mine->done[c], d->done[c]), "ipc event");
      mine->device = ctx->device;
      mine->pid = static_cast<int>(getpid());
      d->rv->barrier();  // every slot written
      for (int r = 0; r < d->world; ++r) {
        if (r == rank) continue;
        DistSlot* ps = static_cast<DistSlot*>(d->rv->slot(r));
        ck(cudaIpcOpenMemHandle(&d->peer_re[r], ps->re, cudaIpcMemLazyEnablePeerAccess), "open peer re");
        ck(cudaIpcOpenMemHandle(&d->peer_im[r], ps->im, cudaIpcMemLazyEnablePeerAccess), "open peer im");
        ck(cudaIpcOpenEventHandle(&d->peer_ready[r], ps->ready), "open peer event");
        for (int c = 0; c < (1 << kMaxPipelineBits); ++c)
          ck(cudaIpcOpenEventHandle(&d->peer_done[r][c], ps->done[c]), "open peer event");
      }
      d->rv->barrier();  // every rank mapped its peers
    }
    *out = d.release();
  })
}

int tsg_dist_destroy(tsg_dist* d) {
  if (!d) return TSG_OK;
  cudaSetDevice(d->ctx->device);
  cudaStreamSynchronize(d->st->stream);
  cudaStreamSynchronize(d->comm);
  d->prepared.clear();
  // peers may still read or write this shard until they are done with the
  // last exchange: meet them before unmapping and freeing
  try {
    if (d->world > 1) d->rv->barrier();
  } catch (...) {
  }
  for (int r = 0; r < d->world; ++r) {
    if (r == d->rank) continue;
    if (d->peer_re[r]) cudaIpcCloseMemHandle(d->peer_re[r]);
    if (d->peer_im[r]) cudaIpcCloseMemHandle(d->peer_im[r]);
    if (d->peer_ready[r]) cudaEventDestroy(d->peer_ready[r]);
    for (cudaEvent_t e : d->peer_done[r])
      if (e) cudaEventDestroy(e);
  }
  try {
    if (d->world > 1) d->rv->barrier();
  } catch (...) {
  }
  for (cudaEvent_t e : d->xt) cudaEventDestroy(e);
  for (cudaEvent_t e : {d->e0, d->e1, d->ready})
    if (e) cudaEventDestroy(e);
  for (cudaEvent_t e : d->done)
    if (e) cudaEventDestroy(e);
  if (d->comm) cudaStreamDestroy(d->comm);
  tsg_state_destroy(d->st);
  delete d;
  return TSG_OK;
}

int tsg_dist_init_basis(tsg_dist* d, uint64_t x) {
  TSG_TRY({
    require(d != nullptr, "null handle");
    const int nl = d->n - d->n_global;
    require(x < (uint64_t{1} << d->n), "basis index out of range");
    if (static_cast<int>(x >> nl) == d->rank) {
      if (tsg_state_init_basis(d->st, x & ((uint64_t{1} << nl) - 1))) throw SimError(tsg_last_error());
    } else {
      const size_t bytes = d->st->size() * d->st->amp_bytes();
      ck(cudaMemsetAsync(d->st->re, 0, bytes, d->st->stream), "memset");
      ck(cudaMemsetAsync(d->st->im, 0, bytes, d->st->stream), "memset");
    }
  })
}

int tsg_dist_upload_local(tsg_dist* d, const double* re, const double* im) {
  if (!d) {
    tsg_detail::set_error("null handle");
    return TSG_ERR_CONFIG;
  }
  return tsg_state_upload(d->st, re, im);
}

// local_only != 0: the segments alone, exchanges skipped (the compute-only
// timeline the exposed swap time is measured against; leaves the state wrong)
static int dist_run_impl(tsg_dist* d, const tsc_shard_plan* plan, int local_only, tsg_run_report* report) {
  TSG_TRY({
    require(d && plan, "null argument");
    const ShardPlan& sp = plan->plan;
    require(sp.n == d->n && sp.n_global == d->n_global, "shard plan does not match the distributed state");
    use_device(d->ctx);
    const PreparedRank& pr = prepared_for(d, plan);
    cudaStream_t s = d->st->stream;
    uint64_t exchanged = 0, launches = 0;
    size_t xi = 0;
    ck(cudaEventRecord(d->e0, s), "event");
    for (size_t i = 0; i < pr.items.size(); ++i) {
      const DistItem& it = pr.items[i];
      if (!it.swap) {
        launches += run_segment(it, d->st);
        continue;
      }
      if (local_only) continue;
      const DistItem* next = i + 1 < pr.items.size() ? &pr.items[i + 1] : nullptr;
      bool consumed = false;
      launches += dist_exchange(d, it, next, xi++, &consumed);
      exchanged += it.moved_bytes;
      if (consumed) ++i;
    }
    ck(cudaEventRecord(d->e1, s), "event");
    ck(cudaEventSynchronize(d->e1), "dist sync");
    ck(cudaStreamSynchronize(d->comm), "comm sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, d->e0, d->e1), "elapsed");
    double xs = 0.0;
    for (size_t k = 0; k < xi; ++k) {
      float x = 0.f;
      ck(cudaEventElapsedTime(&x, d->xt[2 * k], d->xt[2 * k + 1]), "elapsed");
      xs += x * 1e-3;
    }
    if (report) {
      *report = tsg_run_report{};
      report->execution_s = ms * 1e-3;
      report->gates = sp.ops.size();
      report->launches = launches;
      report->bytes = 0;
      for (const DistItem& it : pr.items)
        if (!it.swap) report->bytes += it.full->bytes;
      report->exchanged_bytes = exchanged;
      report->exchange_s = xs;
    }
  })
}

int tsg_dist_run(tsg_dist* d, const tsc_shard_plan* plan, tsg_run_report* report) {
  return dist_run_impl(d, plan, 0, report);
}

int tsg_dist_run_local_only(tsg_dist* d, const tsc_shard_plan* plan, tsg_run_report* report) {
  return dist_run_impl(d, plan, 1, report);
}

// Sharded QSV1 (SPEC.md:565 per shard): <path>.r<rank> is a plain QSV1 dump
// of this rank's 2^n_local amplitudes in physical order; rank 0 also writes
// <path>.layout -- n, n_global, precision and the qubit map (logical qubit q
// at physical position pos[q]) the shards are laid out in.  A resumed run
// loads the shards and continues with plans made for the same layout.
int tsg_dist_dump(tsg_dist* d, const char* path, const int* pos) {
  TSG_TRY({
    require(d && path && pos, "null argument");
    std::vector<int> seen(d->n, 0);
    for (int q = 0; q < d->n; ++q) {
      require(pos[q] >= 0 && pos[q] < d->n && !seen[pos[q]], "qubit map is not a permutation");
      seen[pos[q]] = 1;
    }
    const std::string base(path);
    if (tsg_state_dump(d->st, (base + ".r" + std::to_string(d->rank)).c_str())) throw SimError(tsg_last_error());
    if (d->rank == 0) {
      std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen((base + ".layout").c_str(), "w"), std::fclose);
      if (!f) throw SimError("cannot open " + base + ".layout for writing");
      std::fprintf(f.get(), "qsv1-sharded 1\nn %d\nn_global %d\nprecision %d\npos", d->n, d->n_global, d->st->prec);
      for (int q = 0; q < d->n; ++q) std::fprintf(f.get(), " %d", pos[q]);
      std::fprintf(f.get(), "\n");
    }
  })
}

int tsg_dist_load(tsg_dist* d, const char* path, int* pos) {
  TSG_TRY({
    require(d && path && pos, "null argument");
    const std::string base(path);
    std::unique_ptr<FILE, int (*)(FILE*)> f(std::fopen((base + ".layout").c_str(), "r"), std::fclose);
    if (!f) throw SimError("cannot open " + base + ".layout");
    int version = 0, n = 0, g = 0, prec = 0;
    if (std::fscanf(f.get(), "qsv1-sharded %d n %d n_global %d precision %d pos", &version, &n, &g, &prec) != 4 ||
        version != 1)
      throw SimError(base + ".layout: not a sharded QSV1 layout");
    require(n == d->n && g == d->n_global && prec == d->st->prec, "sharded dump does not match the distributed state");
    for (int q = 0; q < n; ++q)
      if (std::fscanf(f.get(), "%d", &pos[q]) != 1) throw SimError(base + ".layout: truncated qubit map");
    if (tsg_state_load(d->st, (base + ".r" + std::to_string(d->rank)).c_str())) throw SimError(tsg_last_error());
  })
}

int tsg_dist_download_local(tsg_dist* d, double* re, double* im) {
  if (!d) {
    tsg_detail::set_error("null handle");
    return TSG_ERR_CONFIG;
  }
  return tsg_state_download(d->st, re, im);
}

int tsg_dist_local_sumsq(tsg_dist* d, double* out) {
  TSG_TRY({
    require(d && out, "null argument");
    use_device(d->ctx);
    const double nrm = state_norm(d->st);
    *out = nrm * nrm;
  })
}

}  // extern "C"
