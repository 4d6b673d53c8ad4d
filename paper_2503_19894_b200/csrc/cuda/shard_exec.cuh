// Sharded execution (include/tilesim/shard.hpp schedules) -- included at the
// end of runtime.cu, whose handle types and launch helpers it shares.
//
//  tsg_vshard_run  2^g virtual shards on one device; a swap is one in-place
//                  kernel over each shard pair (single-GPU emulation of the
//                  distributed path, used by the GPU parity tests)
//  tsg_dist_*      one process per GPU; a swap is a chunked NCCL send/recv of
//                  the half whose local bit differs from the rank bit (the
//                  half is contiguous when the local position is the top bit,
//                  which the planner prefers), packed otherwise
#include <dlfcn.h>
#include <nccl.h>

namespace {

// ------------------------------------------------------------------ kernels
__device__ __forceinline__ uint64_t with_bit(uint64_t i, int b, uint64_t v) {
  const uint64_t low = i & ((uint64_t{1} << b) - 1);
  return ((i >> b) << (b + 1)) | (v << b) | low;
}

// dst[i] = src[with_bit(first + i, b, v)]    (pack a half into contiguous order)
template <typename Real>
__global__ void k_pack_half(const Real* __restrict__ src, Real* __restrict__ dst, uint64_t first, uint64_t count, int b,
                            uint64_t v) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
    dst[i] = src[with_bit(first + i, b, v)];
}

template <typename Real>
__global__ void k_unpack_half(const Real* __restrict__ src, Real* __restrict__ dst, uint64_t first, uint64_t count,
                              int b, uint64_t v) {
  const uint64_t stride = static_cast<uint64_t>(gridDim.x) * blockDim.x;
  for (uint64_t i = static_cast<uint64_t>(blockIdx.x) * blockDim.x + threadIdx.x; i < count; i += stride)
    dst[with_bit(first + i, b, v)] = src[i];
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

// ------------------------------------------------------- prepared schedule
struct PreparedOp {
  bool swap = false;
  bool skip = false;
  // local gates run as programs (tile passes, block splits): the first op of
  // a run of local gates holds the run's program, the others are in_seg
  tsg_program* prog = nullptr;
  bool in_seg = false;
  std::vector<std::pair<int, int>> swaps;
  KernelPlan plan;
  LaunchStructure ls;
  tsg::GateLaunch launch;
  bool has_mat = false;
  size_t mat_off = 0;
};

struct PreparedRank {
  std::vector<PreparedOp> ops;
  void* arena = nullptr;
  ~PreparedRank() {
    if (arena) cudaFree(arena);
    for (PreparedOp& po : ops)
      if (po.prog) tsg_program_destroy(po.prog);
  }
};

std::unique_ptr<PreparedRank> prepare_rank(const ShardPlan& plan, uint64_t rank, int prec, tsg_ctx* ctx) {
  auto pr = std::make_unique<PreparedRank>();
  std::vector<unsigned char> arena;
  const int nl = plan.n_local;
  Circuit seg;  // the open run of local gates (this rank's sub-gates)
  seg.n_qubits = nl;
  size_t seg_first = 0;
  auto close_segment = [&]() {
    if (seg.gates.empty()) return;
    pr->ops[seg_first].prog = build_program(ctx, seg, 1e-8, 1e-8, prec).release();
    seg.gates.clear();
  };
  for (const ShardOp& op : plan.ops) {
    PreparedOp po;
    if (op.kind == ShardOp::Kind::Swap) {
      close_segment();
      po.swap = true;
      po.swaps = op.swaps;
      pr->ops.push_back(std::move(po));
      continue;
    }
    const Gate g = op.kind == ShardOp::Kind::Local ? op.gate : rank_subgate(op, nl, rank);
    if (g.k() == 0) {  // every target global: a rank-wide phase
      close_segment();
      const cplx v = g.matrix.at(0, 0);
      if (v == cplx(1.0, 0.0)) {
        po.skip = true;
      } else {
        po.ls.klass = KernelClass::Diagonal;
        po.ls.ks = 0;
        po.ls.sub_re = {v.real()};
        po.ls.sub_im = {v.imag()};
        po.launch.klass = static_cast<int>(KernelClass::Diagonal);
        po.launch.ks = 0;
        po.launch.n = nl;
        po.launch.full_range = true;
      }
      pr->ops.push_back(std::move(po));
      continue;
    }
    if (seg.gates.empty()) seg_first = pr->ops.size();
    else po.in_seg = true;
    seg.gates.push_back(g);
    pr->ops.push_back(std::move(po));
  }
  close_segment();
  for (PreparedOp& po : pr->ops) {  // pointers into the (now stable) vectors
    po.launch.m_re = po.ls.sub_re.data();
    po.launch.m_im = po.ls.sub_im.data();
  }
  if (!arena.empty()) {
    ck(cudaSetDevice(ctx->device), "cudaSetDevice");
    ck(cudaMalloc(&pr->arena, arena.size()), "cudaMalloc shard arena");
    ck(cudaMemcpy(pr->arena, arena.data(), arena.size(), cudaMemcpyHostToDevice), "shard arena upload");
  }
  return pr;
}

// returns the kernels launched
uint64_t apply_prepared(const PreparedOp& po, const PreparedRank& pr, tsg_state* st) {
  if (po.skip || po.swap || po.in_seg) return 0;
  if (po.prog) {
    run_program(st, po.prog, nullptr);
    return po.prog->launches;
  }
  const int prec = st->prec;
  cudaStream_t s = st->stream;
  const int num_sms = st->ctx->num_sms;
  void* re = st->re;
  void* im = st->im;
  tsg::GateLaunch g = po.launch;
  g.re = re;
  g.im = im;
  if (po.has_mat) g.dev_mat = static_cast<unsigned char*>(pr.arena) + po.mat_off;
  prec == 64 ? tsg::launch_gate_f64(g, s, num_sms) : tsg::launch_gate_f32(g, s, num_sms);
  return 1;
}

// ------------------------------------------------------------ NCCL loader
struct NcclApi {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::string error;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      error = std::string("cannot load libnccl.so.2: ") + dlerror();
      return;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
    api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
    api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
    api.Send = reinterpret_cast<decltype(api.Send)>(sym("ncclSend"));
    api.Recv = reinterpret_cast<decltype(api.Recv)>(sym("ncclRecv"));
    api.GroupStart = reinterpret_cast<decltype(api.GroupStart)>(sym("ncclGroupStart"));
    api.GroupEnd = reinterpret_cast<decltype(api.GroupEnd)>(sym("ncclGroupEnd"));
    api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
    if (!api.GetUniqueId || !api.CommInitRank || !api.Send || !api.Recv || !api.GroupStart || !api.GroupEnd)
      error = "libnccl.so.2 lacks the point-to-point API";
  });
  if (!error.empty()) throw SimError(error);
  return api;
}

void nck(ncclResult_t r, const char* what) {
  if (r != ncclSuccess)
    throw SimError(std::string("NCCL error in ") + what + ": " + (nccl().GetErrorString ? nccl().GetErrorString(r) : "?"));
}

}  // namespace

struct tsg_dist {
  tsg_ctx* ctx = nullptr;
  tsg_state* st = nullptr;  // this rank's 2^n_local shard
  int n = 0, n_global = 0, rank = 0, world = 1;
  ncclComm_t comm = nullptr;
  void* sendbuf = nullptr;  // chunk buffers (one array at a time)
  void* recvbuf = nullptr;
  uint64_t chunk = 0;       // elements per chunk
  std::map<const tsc_shard_plan*, std::unique_ptr<PreparedRank>> prepared;
  cudaEvent_t e0 = nullptr, e1 = nullptr, x0 = nullptr, x1 = nullptr;
};

namespace {

// exchange the half of array `a` whose local bit `lp` equals v with the peer
void exchange_half(tsg_dist* d, void* a, int lp, uint64_t v, int peer) {
  const int nl = d->n - d->n_global;
  const size_t es = d->st->amp_bytes();
  const uint64_t half = uint64_t{1} << (nl - 1);
  const ncclDataType_t dt = es == 8 ? ncclFloat64 : ncclFloat32;
  cudaStream_t s = d->st->stream;
  const bool contiguous = lp == nl - 1;
  unsigned char* base = static_cast<unsigned char*>(a) + (contiguous ? v * half * es : 0);
  for (uint64_t first = 0; first < half; first += d->chunk) {
    const uint64_t cnt = std::min(d->chunk, half - first);
    const void* src = base + first * es;
    if (!contiguous) {
      const unsigned g = ew_grid(d->ctx, cnt);
      if (es == 8) k_pack_half<double><<<g, 256, 0, s>>>((const double*)a, (double*)d->sendbuf, first, cnt, lp, v);
      else k_pack_half<float><<<g, 256, 0, s>>>((const float*)a, (float*)d->sendbuf, first, cnt, lp, v);
      ck(cudaGetLastError(), "k_pack_half");
      src = d->sendbuf;
    }
    nck(nccl().GroupStart(), "group start");
    nck(nccl().Send(src, cnt, dt, peer, d->comm, s), "send");
    nck(nccl().Recv(d->recvbuf, cnt, dt, peer, d->comm, s), "recv");
    nck(nccl().GroupEnd(), "group end");
    if (contiguous) {
      ck(cudaMemcpyAsync(base + first * es, d->recvbuf, cnt * es, cudaMemcpyDeviceToDevice, s), "unpack copy");
    } else {
      const unsigned g = ew_grid(d->ctx, cnt);
      if (es == 8) k_unpack_half<double><<<g, 256, 0, s>>>((const double*)d->recvbuf, (double*)a, first, cnt, lp, v);
      else k_unpack_half<float><<<g, 256, 0, s>>>((const float*)d->recvbuf, (float*)a, first, cnt, lp, v);
      ck(cudaGetLastError(), "k_unpack_half");
    }
  }
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
    // one stream orders every shard's launches and the swaps (the shards'
    // own streams are restored before they are destroyed)
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
    for (size_t i = 0; i < sp.ops.size(); ++i) {
      const ShardOp& op = sp.ops[i];
      if (op.kind == ShardOp::Kind::Swap) {
        for (const auto& sw : op.swaps) {
          const int bit = sw.first - nl, lp = sw.second;
          for (uint64_t s = 0; s < S; ++s) {
            if ((s >> bit) & 1u) continue;
            tsg_state* a = shards[s].get();
            tsg_state* c = shards[s | (uint64_t{1} << bit)].get();
            const uint64_t half = local / 2;
            const unsigned gr = ew_grid(ctx, half);
            if (precision_bits == 64) {
              k_swap_halves<double><<<gr, 256, 0, stream>>>((double*)a->re, (double*)c->re, half, lp);
              k_swap_halves<double><<<gr, 256, 0, stream>>>((double*)a->im, (double*)c->im, half, lp);
            } else {
              k_swap_halves<float><<<gr, 256, 0, stream>>>((float*)a->re, (float*)c->re, half, lp);
              k_swap_halves<float><<<gr, 256, 0, stream>>>((float*)a->im, (float*)c->im, half, lp);
            }
            ck(cudaGetLastError(), "k_swap_halves");
            exchanged += 2 * half * a->amp_bytes();  // per rank, one direction
          }
        }
        continue;
      }
      for (uint64_t s = 0; s < S; ++s) launches += apply_prepared(prep[s]->ops[i], *prep[s], shards[s].get());
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
      report->exchanged_bytes = exchanged / S;
    }
  })
}

int tsg_dist_unique_id(unsigned char id[128]) {
  TSG_TRY({
    require(id != nullptr, "null argument");
    ncclUniqueId uid;
    nck(nccl().GetUniqueId(&uid), "ncclGetUniqueId");
    std::memcpy(id, uid.internal, 128);
  })
}

int tsg_dist_create(tsg_ctx* ctx, int n_qubits, int precision_bits, int n_global, int rank, const unsigned char id[128],
                    tsg_dist** out) {
  TSG_TRY({
    require(ctx && id && out, "null argument");
    require(n_global >= 0 && n_global < n_qubits, "n_global must be in [0, n)");
    require(rank >= 0 && rank < (1 << n_global), "rank out of range");
    use_device(ctx);
    auto d = std::make_unique<tsg_dist>();
    d->ctx = ctx;
    d->n = n_qubits;
    d->n_global = n_global;
    d->rank = rank;
    d->world = 1 << n_global;
    if (tsg_state_create(ctx, n_qubits - n_global, precision_bits, &d->st)) throw SimError(tsg_last_error());
    if (d->world > 1) {
      ncclUniqueId uid;
      std::memcpy(uid.internal, id, 128);
      nck(nccl().CommInitRank(&d->comm, d->world, uid, rank), "ncclCommInitRank");
    }
    const uint64_t half = uint64_t{1} << std::max(0, n_qubits - n_global - 1);
    d->chunk = std::min<uint64_t>(half, uint64_t{1} << 26);
    const size_t bytes = d->chunk * d->st->amp_bytes();
    ck(cudaMalloc(&d->sendbuf, bytes), "cudaMalloc sendbuf");
    ck(cudaMalloc(&d->recvbuf, bytes), "cudaMalloc recvbuf");
    for (cudaEvent_t* e : {&d->e0, &d->e1, &d->x0, &d->x1}) ck(cudaEventCreate(e), "event");
    *out = d.release();
  })
}

int tsg_dist_destroy(tsg_dist* d) {
  if (!d) return TSG_OK;
  cudaSetDevice(d->ctx->device);
  d->prepared.clear();
  if (d->comm && nccl().CommDestroy) nccl().CommDestroy(d->comm);
  cudaFree(d->sendbuf);
  cudaFree(d->recvbuf);
  for (cudaEvent_t e : {d->e0, d->e1, d->x0, d->x1})
    if (e) cudaEventDestroy(e);
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

int tsg_dist_run(tsg_dist* d, const tsc_shard_plan* plan, tsg_run_report* report) {
  TSG_TRY({
    require(d && plan, "null argument");
    const ShardPlan& sp = plan->plan;
    require(sp.n == d->n && sp.n_global == d->n_global, "shard plan does not match the distributed state");
    use_device(d->ctx);
    auto it = d->prepared.find(plan);
    if (it == d->prepared.end())
      it = d->prepared.emplace(plan, prepare_rank(sp, d->rank, d->st->prec, d->ctx)).first;
    const PreparedRank& pr = *it->second;
    const int nl = sp.n_local;
    cudaStream_t s = d->st->stream;
    uint64_t exchanged = 0, launches = 0;
    double xs = 0.0;
    ck(cudaEventRecord(d->e0, s), "event");
    for (size_t i = 0; i < sp.ops.size(); ++i) {
      const PreparedOp& po = pr.ops[i];
      if (!po.swap) {
        launches += apply_prepared(po, pr, d->st);
        continue;
      }
      ck(cudaEventRecord(d->x0, s), "event");
      for (const auto& sw : po.swaps) {
        const int bit = sw.first - nl, lp = sw.second;
        const int peer = d->rank ^ (1 << bit);
        const uint64_t v = 1 - ((static_cast<uint64_t>(d->rank) >> bit) & 1u);  // the half this rank sends
        exchange_half(d, d->st->re, lp, v, peer);
        exchange_half(d, d->st->im, lp, v, peer);
        exchanged += 2 * (d->st->size() / 2) * d->st->amp_bytes();
      }
      ck(cudaEventRecord(d->x1, s), "event");
      ck(cudaEventSynchronize(d->x1), "exchange sync");
      float ms = 0.f;
      ck(cudaEventElapsedTime(&ms, d->x0, d->x1), "elapsed");
      xs += ms * 1e-3;
    }
    ck(cudaEventRecord(d->e1, s), "event");
    ck(cudaEventSynchronize(d->e1), "dist sync");
    float ms = 0.f;
    ck(cudaEventElapsedTime(&ms, d->e0, d->e1), "elapsed");
    if (report) {
      *report = tsg_run_report{};
      report->execution_s = ms * 1e-3;
      report->gates = sp.ops.size();
      report->launches = launches;
      report->bytes = launches * 2 * d->st->size() * d->st->amp_bytes() * 2;
      report->exchanged_bytes = exchanged;
      report->exchange_s = xs;
    }
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
