// shard.cu -- multi-GPU IMM: the exchange step.
//
// Slot j's set depends only on (run_seed, j) (sampling.hpp:179), so a top-up of
// `count` new slots splits into N contiguous shards and rank r samples shard r
// with no communication. The one real exchange is assembling the collection:
// every rank broadcasts its shard -- the flat member lists, their offsets, the
// set -> row map and the dense rows -- straight from device memory over NCCL
// (one ncclBroadcast per array and rank, grouped), and every rank appends the N
// shards in rank order, which is slot order. Each rank then holds exactly the
// reference's collection and its fused counter (the append recounts the new
// sets on the device: Sigma |R| atomics, less than an n-entry AllReduce at IMM
// sizes), so the k-round selection runs replicated with identical results and
// no further traffic; the IMM decisions (theta, LB) are the same on every rank.
//
// NCCL is loaded at first use (dlopen libnccl.so.2 -- the process's copy when
// torch already loaded one), so single-GPU users of librrgpu.so never map it.
#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <stdexcept>
#include <type_traits>
#include <string>
#include <vector>

#include "internal.hpp"

namespace rrgpu {

namespace {

// the NCCL subset used here (nccl.h ABI: enums as int, opaque comm pointer)
typedef struct { char internal[128]; } NcclUniqueId;
typedef void* NcclComm;
typedef int NcclResult;
constexpr int kNcclUint8 = 1, kNcclUint32 = 3, kNcclUint64 = 5;

struct Nccl {
  NcclResult (*get_unique_id)(NcclUniqueId*) = nullptr;
  NcclResult (*comm_init_rank)(NcclComm*, int, NcclUniqueId, int) = nullptr;
  NcclResult (*comm_destroy)(NcclComm) = nullptr;
  NcclResult (*comm_count)(NcclComm, int*) = nullptr;
  NcclResult (*comm_user_rank)(NcclComm, int*) = nullptr;
  NcclResult (*broadcast)(const void*, void*, size_t, int, int, NcclComm, cudaStream_t) = nullptr;
  NcclResult (*all_gather)(const void*, void*, size_t, int, NcclComm, cudaStream_t) = nullptr;
  NcclResult (*group_start)() = nullptr;
  NcclResult (*group_end)() = nullptr;
  const char* (*error_string)(NcclResult) = nullptr;
  bool ok = false;
  std::string why;
};

const Nccl& nccl() {
  static Nccl n;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      n.why = std::string("libnccl.so.2 not found: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      if (!fn) n.why += std::string(n.why.empty() ? "" : ", ") + name;
    };
    sym(n.get_unique_id, "ncclGetUniqueId");
    sym(n.comm_init_rank, "ncclCommInitRank");
    sym(n.comm_destroy, "ncclCommDestroy");
    sym(n.comm_count, "ncclCommCount");
    sym(n.comm_user_rank, "ncclCommUserRank");
    sym(n.broadcast, "ncclBroadcast");
    sym(n.all_gather, "ncclAllGather");
    sym(n.group_start, "ncclGroupStart");
    sym(n.group_end, "ncclGroupEnd");
    sym(n.error_string, "ncclGetErrorString");
    n.ok = n.why.empty();
    if (!n.ok) n.why = "missing NCCL symbols: " + n.why;
  });
  return n;
}

void nccl_check(NcclResult r, const char* what) {
  if (r != 0) {
    const Nccl& n = nccl();
    throw std::runtime_error(std::string(what) + ": " + (n.error_string ? n.error_string(r) : "?"));
  }
}

}  // namespace

bool nccl_available(std::string* why) {
  const Nccl& n = nccl();
  if (!n.ok && why) *why = n.why;
  return n.ok;
}

void nccl_unique_id(uint8_t out[128]) {
  const Nccl& n = nccl();
  if (!n.ok) throw std::runtime_error(n.why);
  NcclUniqueId id;
  nccl_check(n.get_unique_id(&id), "ncclGetUniqueId");
  std::memcpy(out, id.internal, 128);
}

void* nccl_comm_create(const uint8_t id[128], int nranks, int rank) {
  const Nccl& n = nccl();
  if (!n.ok) throw std::runtime_error(n.why);
  NcclUniqueId uid;
  std::memcpy(uid.internal, id, 128);
  NcclComm c = nullptr;
  nccl_check(n.comm_init_rank(&c, nranks, uid, rank), "ncclCommInitRank");
  return c;
}

void nccl_comm_destroy(void* comm) {
  const Nccl& n = nccl();
  if (n.ok && comm) n.comm_destroy(static_cast<NcclComm>(comm));
}

void nccl_comm_shape(void* comm, int* nranks, int* rank) {
  const Nccl& n = nccl();
  if (!n.ok) throw std::runtime_error(n.why);
  nccl_check(n.comm_count(static_cast<NcclComm>(comm), nranks), "ncclCommCount");
  nccl_check(n.comm_user_rank(static_cast<NcclComm>(comm), rank), "ncclCommUserRank");
}

// Shard r's arrays in device memory (rank r's side store, or what rank r broadcast).
struct Shard {
  uint64_t nsets = 0, total = 0, ndense = 0;
  DevBuf<uint64_t> off;   // nsets + 1, relative
  DevBuf<uint32_t> mem;   // total
  DevBuf<uint32_t> dix;   // nsets (rows relative to the shard)
  DevBuf<uint32_t> dbits; // ndense x dwords
  DevBuf<uint32_t> dlen, droot;
};

rrg_status append_shards(rrg_store* dst, std::vector<Shard>& shards);

// Exchanges the side store of this rank (its shard) with every other rank over
// `comm` and appends all shards, in rank order, to `dst`.
rrg_status exchange_impl(rrg_store* side, rrg_store* dst, void* comm);

rrg_status exchange_and_append(rrg_store* side, rrg_store* dst, void* comm) {
  try {
    return exchange_impl(side, dst, comm);
  } catch (const CudaError& e) {
    set_error(std::string(e.where) + ": " + cudaGetErrorString(e.err));
    return e.err == cudaErrorMemoryAllocation ? RRG_ENOMEM : RRG_ECUDA;
  } catch (const std::exception& e) {
    set_error(e.what());
    return RRG_ECUDA;
  }
}

rrg_status exchange_impl(rrg_store* side, rrg_store* dst, void* comm) {
  const Nccl& n = nccl();
  if (!n.ok) throw std::runtime_error(n.why);
  rrg_graph* g = dst->g;
  const cudaStream_t st = g->stream;
  NcclComm c = static_cast<NcclComm>(comm);
  int nranks = 1, rank = 0;
  nccl_comm_shape(comm, &nranks, &rank);
  // shard sizes: one AllGather of 3 u64 per rank
  DevBuf<uint64_t> hdr, hdrs;
  hdr.reserve_discard(4);
  hdrs.reserve_discard(4ull * nranks);
  const uint64_t mine[4] = {side->nsets, side->total, side->ndense, 0};
  RRG_CUDA(cudaMemcpyAsync(hdr.ptr, mine, sizeof(mine), cudaMemcpyHostToDevice, st));
  nccl_check(n.all_gather(hdr.ptr, hdrs.ptr, 4, kNcclUint64, c, st), "ncclAllGather");
  std::vector<uint64_t> h(4ull * nranks);
  RRG_CUDA(cudaMemcpyAsync(h.data(), hdrs.ptr, h.size() * 8, cudaMemcpyDeviceToHost, st));
  host_sync((st));
  std::vector<Shard> shards(nranks);
  const uint32_t W = dst->dwords;
  for (int r = 0; r < nranks; ++r) {
    Shard& s = shards[r];
    s.nsets = h[4 * r];
    s.total = h[4 * r + 1];
    s.ndense = h[4 * r + 2];
    s.off.reserve_discard(s.nsets + 1);
    s.mem.reserve_discard(s.total ? s.total : 1);
    s.dix.reserve_discard(s.nsets ? s.nsets : 1);
    s.dbits.reserve_discard(s.ndense ? s.ndense * W : 1);
    s.dlen.reserve_discard(s.ndense ? s.ndense : 1);
    s.droot.reserve_discard(s.ndense ? s.ndense : 1);
  }
  // the root's own arrays are the send buffers (its side store is compact:
  // offsets from 0, rows [0, ndense))
  nccl_check(n.group_start(), "ncclGroupStart");
  for (int r = 0; r < nranks; ++r) {
    Shard& s = shards[r];
    const bool root = r == rank;
    auto bc = [&](const void* send, void* recv, size_t count, int type) {
      if (count) nccl_check(n.broadcast(root ? send : recv, recv, count, type, r, c, st),
                            "ncclBroadcast");
    };
    bc(side->off.ptr, s.off.ptr, s.nsets + 1, kNcclUint64);
    bc(side->mem.ptr, s.mem.ptr, s.total, kNcclUint32);
    bc(side->dix.ptr, s.dix.ptr, s.nsets, kNcclUint32);
    bc(side->dbits.ptr, s.dbits.ptr, s.ndense * W, kNcclUint32);
    bc(side->dlen.ptr, s.dlen.ptr, s.ndense, kNcclUint32);
    bc(side->droot.ptr, s.droot.ptr, s.ndense, kNcclUint32);
  }
  nccl_check(n.group_end(), "ncclGroupEnd");
  return append_shards(dst, shards);
}

// Appends `shards` in order to `dst`, each through a view store that borrows the
// shard's buffers, so rrg_store_append_from does the copies, the row gathers
// and the recount of the new sets.
rrg_status append_shards(rrg_store* dst, std::vector<Shard>& shards) {
  rrg_graph* g = dst->g;
  for (Shard& s : shards) {
    if (!s.nsets) continue;
    // a view store over the shard's buffers (not owned: released before return)
    rrg_store view;
    view.g = g;
    view.nsets = s.nsets;
    view.total = s.total;
    view.ndense = s.ndense;
    view.dwords = dst->dwords;
    auto borrow = [](auto& to, auto& from, size_t cap) {
      to.ptr = from.ptr;
      to.cap = cap;
      to.bytes = 0;
    };
    borrow(view.off, s.off, s.nsets + 1);
    borrow(view.mem, s.mem, s.total);
    borrow(view.dix, s.dix, s.nsets);
    borrow(view.dbits, s.dbits, s.ndense * dst->dwords);
    borrow(view.dlen, s.dlen, s.ndense);
    borrow(view.droot, s.droot, s.ndense);
    const rrg_status r = rrg_store_append_from(dst, &view, 0, s.nsets);
    // the view's buffers are the shard's: drop them before its destructor runs
    view.off.ptr = nullptr;
    view.mem.ptr = view.dix.ptr = view.dbits.ptr = view.dlen.ptr = view.droot.ptr = nullptr;
    view.off.cap = view.mem.cap = view.dix.cap = view.dbits.cap = view.dlen.cap = view.droot.cap = 0;
    if (r != RRG_OK) return r;
  }
  return RRG_OK;
}

}  // namespace rrgpu

extern "C" {

rrg_status rrg_nccl_unique_id(uint8_t* id) {
  if (!id) {
    rrgpu::set_error("null argument");
    return RRG_EINVAL;
  }
  try {
    rrgpu::nccl_unique_id(id);
    return RRG_OK;
  } catch (const std::exception& e) {
    rrgpu::set_error(e.what());
    return RRG_ECUDA;
  }
}

rrg_status rrg_nccl_comm_create(const uint8_t* id, int nranks, int rank, void** comm) {
  if (!id || !comm || nranks < 1 || rank < 0 || rank >= nranks) {
    rrgpu::set_error("nccl_comm_create: bad argument");
    return RRG_EINVAL;
  }
  try {
    *comm = rrgpu::nccl_comm_create(id, nranks, rank);
    return RRG_OK;
  } catch (const std::exception& e) {
    rrgpu::set_error(e.what());
    return RRG_ECUDA;
  }
}

void rrg_nccl_comm_destroy(void* comm) { rrgpu::nccl_comm_destroy(comm); }

}  // extern "C"
