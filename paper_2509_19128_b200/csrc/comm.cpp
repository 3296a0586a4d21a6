// comm.cpp -- the weight-transfer channel and the trainer's gradient
// all-reduce over NCCL (NVLink / NVSwitch on one node), behind the C ABI so a
// C++ host drives them without Python (include/streamrl_b200.h, srl_comm_*).
//
// The reference pushes the whole policy as JSON over HTTP to each member of a
// process group in turn (request_group_weight_update, protocol.cpp:397-406;
// init_process_group, protocol.cpp:378-395; engine.cpp:276-291).  Here one
// collective moves the flat bf16 weight buffer: the trainer root broadcasts
// it straight into every generator engine's standby buffer on a dedicated
// stream while the generator keeps decoding on its own stream, and the
// generator swaps it in at the next token boundary (commit).  Versions stay
// strictly sequential (engine.cpp:82-87): a generator whose engine rejects
// the version still joins the collective (receiving into scratch), so the
// other ranks never hang, and keeps serving at its old version.
//
// NCCL is loaded at run time (dlopen "libnccl.so.2"): the library loads on a
// host without NCCL (the entry points then fail with SRL_NCCL_ERROR), and in
// a process where torch already loaded its NCCL the same copy is shared.
#include <dlfcn.h>
#include <nccl.h>

#include <chrono>
#include <cstring>
#include <mutex>
#include <string>

#include "capi_handles.hpp"

namespace {

struct NcclApi {
  bool ok = false;
  std::string why;
  ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
  ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
  ncclResult_t (*broadcast)(const void*, void*, size_t, ncclDataType_t, int, ncclComm_t,
                            cudaStream_t) = nullptr;
  ncclResult_t (*all_reduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                             cudaStream_t) = nullptr;
  const char* (*error_string)(ncclResult_t) = nullptr;
};

const NcclApi& nccl() {
  static NcclApi api;
  static std::once_flag once;
  std::call_once(once, [] {
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      api.why = std::string("libnccl.so.2 not loadable: ") + dlerror();
      return;
    }
    auto sym = [&](auto& fn, const char* name) {
      fn = reinterpret_cast<std::remove_reference_t<decltype(fn)>>(dlsym(h, name));
      return fn != nullptr;
    };
    api.ok = sym(api.get_unique_id, "ncclGetUniqueId") && sym(api.comm_init_rank, "ncclCommInitRank") &&
             sym(api.comm_destroy, "ncclCommDestroy") && sym(api.broadcast, "ncclBroadcast") &&
             sym(api.all_reduce, "ncclAllReduce") && sym(api.error_string, "ncclGetErrorString");
    if (!api.ok) api.why = "libnccl.so.2 lacks an entry point";
  });
  return api;
}

int nccl_fail(ncclResult_t r, const char* where) {
  return srl::fail(SRL_NCCL_ERROR, std::string(where) + ": " + nccl().error_string(r));
}

#define SRL_NCCL(expr)                                 \
  do {                                                 \
    const ncclResult_t _r = (expr);                    \
    if (_r != ncclSuccess) return nccl_fail(_r, #expr); \
  } while (0)

}  // namespace

struct srl_comm {
  ncclComm_t comm = nullptr;
  int world = 0, rank = 0, device = 0;
  cudaStream_t stream = nullptr;   // the transfer stream (never the decode stream)
  cudaEvent_t begin = nullptr, done = nullptr;
  void* scratch = nullptr;         // receive buffer of a rank whose engine rejected the version
  size_t scratch_bytes = 0;
  bool pending = false;            // a broadcast is in flight
  bool staged = false;             // ... into an engine's standby buffer
  ~srl_comm() {
    if (stream) cudaStreamSynchronize(stream);
    if (comm) nccl().comm_destroy(comm);
    if (scratch) cudaFree(scratch);
    if (begin) cudaEventDestroy(begin);
    if (done) cudaEventDestroy(done);
    if (stream) cudaStreamDestroy(stream);
  }
};

using namespace srl;

extern "C" int srl_comm_unique_id(uint8_t* id_out) {
  if (!id_out) return fail(SRL_INVALID_ARGUMENT, "comm_unique_id: null");
  const NcclApi& n = nccl();
  if (!n.ok) return fail(SRL_NCCL_ERROR, n.why);
  ncclUniqueId id;
  SRL_NCCL(n.get_unique_id(&id));
  std::memcpy(id_out, id.internal, sizeof(id.internal));
  return SRL_OK;
}

extern "C" int srl_comm_init(const uint8_t* id, int32_t world, int32_t rank, int32_t device,
                             srl_comm** out) {
  if (!id || !out || world < 1 || rank < 0 || rank >= world)
    return fail(SRL_INVALID_ARGUMENT, "comm_init: bad arguments");
  const NcclApi& n = nccl();
  if (!n.ok) return fail(SRL_NCCL_ERROR, n.why);
  int count = 0;
  if (cudaGetDeviceCount(&count) != cudaSuccess || count == 0)
    return fail(SRL_NO_DEVICE, "no CUDA device visible");
  if (device < 0 || device >= count) return fail(SRL_INVALID_ARGUMENT, "device index out of range");
  SRL_CUDA(cudaSetDevice(device));
  auto c = std::make_unique<srl_comm>();
  c->world = world;
  c->rank = rank;
  c->device = device;
  SRL_CUDA(cudaStreamCreateWithFlags(&c->stream, cudaStreamNonBlocking));
  SRL_CUDA(cudaEventCreate(&c->begin));
  SRL_CUDA(cudaEventCreate(&c->done));
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, sizeof(uid.internal));
  SRL_NCCL(n.comm_init_rank(&c->comm, world, uid, rank));
  *out = c.release();
  return SRL_OK;
}

extern "C" void srl_comm_destroy(srl_comm* c) { delete c; }

extern "C" int srl_comm_size(const srl_comm* c, int32_t* world, int32_t* rank) {
  if (!c) return fail(SRL_INVALID_ARGUMENT, "comm_size: null");
  if (world) *world = c->world;
  if (rank) *rank = c->rank;
  return SRL_OK;
}

// Plain in-place broadcast of a device buffer (synchronous).
extern "C" int srl_comm_broadcast_bytes(srl_comm* c, int32_t root, void* device_buf, size_t nbytes) {
  if (!c || !device_buf || root < 0 || root >= c->world) return fail(SRL_INVALID_ARGUMENT, "broadcast_bytes");
  SRL_CUDA(cudaSetDevice(c->device));
  SRL_NCCL(nccl().broadcast(device_buf, device_buf, nbytes, ncclUint8, root, c->comm, c->stream));
  SRL_CUDA(cudaStreamSynchronize(c->stream));
  return SRL_OK;
}

// Root side of the group weight push: the trainer's bf16 weights, ordered
// after the trainer's queued work (its last Adam step).  Asynchronous: the
// trainer's stream waits for the send before it touches the weights again.
extern "C" int srl_comm_send_weights(srl_comm* c, srl_trainer* t) {
  if (!c || !t) return fail(SRL_INVALID_ARGUMENT, "send_weights: null");
  if (c->pending) return fail(SRL_BUSY, "a broadcast is already in flight");
  DecoderTrainer& tr = *t->t;
  if (tr.device() != c->device) return fail(SRL_INVALID_ARGUMENT, "trainer and comm on different devices");
  SRL_CUDA(cudaSetDevice(c->device));
  void* w = tr.weights().w;
  const size_t nbytes = tr.weights().bytes;
  SRL_CUDA(cudaEventRecord(c->begin, tr.stream()));
  SRL_CUDA(cudaStreamWaitEvent(c->stream, c->begin, 0));
  SRL_CUDA(cudaEventRecord(c->begin, c->stream));
  SRL_NCCL(nccl().broadcast(w, w, nbytes, ncclUint8, c->rank, c->comm, c->stream));
  SRL_CUDA(cudaEventRecord(c->done, c->stream));
  SRL_CUDA(cudaStreamWaitEvent(tr.stream(), c->done, 0));  // next Adam waits for the send
  c->pending = true;
  c->staged = false;
  return SRL_OK;
}

// Receiver side, part 1: stage new_version in the engine and enqueue the
// receive into its standby buffer; returns at once (decode continues).
// *staged = 0 when the engine rejected the version (version_conflict): the
// rank still receives (into scratch) so the collective completes everywhere.
extern "C" int srl_comm_recv_weights_begin(srl_comm* c, int32_t root, srl_engine* e, int32_t new_version,
                                           int32_t* staged) {
  if (!c || !e || root < 0 || root >= c->world || root == c->rank)
    return fail(SRL_INVALID_ARGUMENT, "recv_weights_begin: bad arguments");
  if (c->pending) return fail(SRL_BUSY, "a broadcast is already in flight");
  if (e->e->device() != c->device) return fail(SRL_INVALID_ARGUMENT, "engine and comm on different devices");
  SRL_CUDA(cudaSetDevice(c->device));
  void* buf = nullptr;
  size_t nbytes = 0;
  int st = e->e->standby_bytes(&nbytes);
  if (st != SRL_OK) return st;
  st = e->e->begin_weight_update(new_version, &buf, &nbytes);
  const bool ok = st == SRL_OK;
  if (!ok) {
    if (st != SRL_VERSION_CONFLICT && st != SRL_BUSY) return st;
    if (c->scratch_bytes < nbytes) {
      if (c->scratch) cudaFree(c->scratch);
      c->scratch = nullptr;
      c->scratch_bytes = 0;
      SRL_CUDA(cudaMalloc(&c->scratch, nbytes));
      c->scratch_bytes = nbytes;
    }
    buf = c->scratch;
  }
  SRL_CUDA(cudaEventRecord(c->begin, c->stream));
  const ncclResult_t r = nccl().broadcast(buf, buf, nbytes, ncclUint8, root, c->comm, c->stream);
  if (r != ncclSuccess) {
    if (ok) e->e->abort_weight_update();
    return nccl_fail(r, "ncclBroadcast");
  }
  SRL_CUDA(cudaEventRecord(c->done, c->stream));
  c->pending = true;
  c->staged = ok;
  if (staged) *staged = ok ? 1 : 0;
  return SRL_OK;
}

// Completion of the in-flight broadcast on any rank (root or receiver):
// waits for the transfer, reports its device time.
extern "C" int srl_comm_wait(srl_comm* c, double* transfer_ms) {
  if (!c) return fail(SRL_INVALID_ARGUMENT, "comm_wait: null");
  if (!c->pending) return fail(SRL_LOGIC_ERROR, "no broadcast in flight");
  SRL_CUDA(cudaEventSynchronize(c->done));
  float ms = 0.0f;
  SRL_CUDA(cudaEventElapsedTime(&ms, c->begin, c->done));
  if (transfer_ms) *transfer_ms = ms;
  c->pending = false;
  return SRL_OK;
}

// Receiver side, part 2: wait for the transfer, then swap the weights in at
// the next token boundary (srl_engine_commit_weight_update).  *applied = 0
// when the engine had rejected the version at begin.
extern "C" int srl_comm_recv_weights_finish(srl_comm* c, srl_engine* e, int32_t new_version,
                                            int32_t* applied, int32_t* version_out,
                                            double* transfer_ms, double* pause_ms) {
  if (!c || !e) return fail(SRL_INVALID_ARGUMENT, "recv_weights_finish: null");
  const bool staged = c->staged;
  int st = srl_comm_wait(c, transfer_ms);
  if (st != SRL_OK) return st;
  c->staged = false;
  int v = 0;
  double ms = 0.0;
  if (!staged) {
    v = e->e->weight_version();
    if (applied) *applied = 0;
  } else {
    st = e->e->commit_weight_update(new_version, &v, &ms);
    if (st != SRL_OK && st != SRL_VERSION_CONFLICT) return st;
    if (applied) *applied = st == SRL_OK ? 1 : 0;
  }
  if (version_out) *version_out = v;
  if (pause_ms) *pause_ms = ms;
  return SRL_OK;
}

// Trainer data parallelism: in-place SUM of the fp32 gradient over the
// trainer group, ordered on the trainer's stream (after the backward, before
// Adam) -- nothing else touches the gradient in between.
extern "C" int srl_comm_allreduce_gradient(srl_comm* c, srl_trainer* t) {
  if (!c || !t) return fail(SRL_INVALID_ARGUMENT, "allreduce_gradient: null");
  DecoderTrainer& tr = *t->t;
  if (tr.device() != c->device) return fail(SRL_INVALID_ARGUMENT, "trainer and comm on different devices");
  SRL_CUDA(cudaSetDevice(c->device));
  SRL_NCCL(nccl().all_reduce(tr.gradient(), tr.gradient(), tr.elements(), ncclFloat32, ncclSum, c->comm,
                             tr.stream()));
  return SRL_OK;
}
