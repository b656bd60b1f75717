// exchange.cpp -- the compressed embedding all-to-all over NCCL (include/embc_cuda.h,
// "compressed embedding all-to-all").  Host orchestration only: the codec runs
// through the library's own C ABI (embc_encode / embc_decode on two contexts),
// the transport is NCCL grouped send/recv, resolved at run time from
// libnccl.so.2 (the copy torch already loaded, or the system one).
//
// Reference: Simulator::rank_body (commsim.hpp:286-435) -- stage 1 compress
// per destination + pack + metadata, stage 2/3 metadata then payload visible to
// the peers, stage 4 decode what this rank receives; byte accounting as
// commsim.hpp:322-353.  Layout for several tables per rank: SURVEY.md App. D.1.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cstdio>
#include <cstring>
#include <functional>
#include <string>
#include <vector>

#include "../../include/embc_cuda.h"

namespace embc_p2p {  // p2p.cu
cudaError_t bump(uint64_t* ctr, cudaStream_t s);
cudaError_t signal(uint64_t* const* d_dst, uint32_t n, const uint64_t* ctr, cudaStream_t s);
cudaError_t wait(const uint64_t* flags, uint32_t n, const uint64_t* ctr, uint64_t minus, uint32_t* timeout,
                 cudaStream_t s);
}  // namespace embc_p2p

namespace {

// ---- NCCL, resolved at run time ----------------------------------------------
struct Nccl {
  ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
  ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
  ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
  ncclResult_t (*GroupStart)() = nullptr;
  ncclResult_t (*GroupEnd)() = nullptr;
  ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
  const char* (*GetErrorString)(ncclResult_t) = nullptr;
  bool ok = false;
  std::string why;
};

const Nccl& nccl() {
  static Nccl n = [] {
    Nccl x;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
      x.why = std::string("cannot load libnccl.so.2: ") + dlerror();
      return x;
    }
    auto sym = [&](const char* name) { return dlsym(h, name); };
    x.GetUniqueId = reinterpret_cast<decltype(x.GetUniqueId)>(sym("ncclGetUniqueId"));
    x.CommInitRank = reinterpret_cast<decltype(x.CommInitRank)>(sym("ncclCommInitRank"));
    x.CommDestroy = reinterpret_cast<decltype(x.CommDestroy)>(sym("ncclCommDestroy"));
    x.GroupStart = reinterpret_cast<decltype(x.GroupStart)>(sym("ncclGroupStart"));
    x.GroupEnd = reinterpret_cast<decltype(x.GroupEnd)>(sym("ncclGroupEnd"));
    x.Send = reinterpret_cast<decltype(x.Send)>(sym("ncclSend"));
    x.Recv = reinterpret_cast<decltype(x.Recv)>(sym("ncclRecv"));
    x.GetErrorString = reinterpret_cast<decltype(x.GetErrorString)>(sym("ncclGetErrorString"));
    x.ok = x.GetUniqueId && x.CommInitRank && x.CommDestroy && x.GroupStart && x.GroupEnd && x.Send &&
           x.Recv && x.GetErrorString;
    if (!x.ok) x.why = "libnccl.so.2 lacks the send/recv API";
    return x;
  }();
  return n;
}

constexpr size_t kMeta = 25;  // ChunkMetadata::kWireSize (container.hpp:193)

struct DevBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFree(p);
    p = nullptr;
    cap = 0;
    const size_t c = std::max<size_t>(bytes, 256);
    cudaError_t e = cudaMalloc(&p, c);
    if (e == cudaSuccess) cap = c;
    return e;
  }
  ~DevBuf() {
    if (p) cudaFree(p);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

struct HostBuf {
  void* p = nullptr;
  size_t cap = 0;
  cudaError_t reserve(size_t bytes) {
    if (bytes <= cap) return cudaSuccess;
    if (p) cudaFreeHost(p);
    p = nullptr;
    cap = 0;
    const size_t c = std::max<size_t>(bytes, 4096);
    cudaError_t e = cudaMallocHost(&p, c);
    if (e == cudaSuccess) cap = c;
    return e;
  }
  ~HostBuf() {
    if (p) cudaFreeHost(p);
  }
  template <typename T>
  T* as() const { return static_cast<T*>(p); }
};

// One table group's buffers (kept across calls; grown, never shrunk).
struct Group {
  DevBuf send, lens, meta, meta_recv, recv;
  HostBuf host;  // lens (u64 x jobs) | metadata records received
  cudaEvent_t encoded = nullptr, arrived = nullptr;
};

// A chunk this rank compresses: table t's rows for destination dst.
struct SendJob {
  uint32_t table, dst;
  const float* src;
};
// A chunk this rank receives: from src, decoded into out ([count, dim]).
struct RecvChunk {
  uint32_t table, src;
  float* out;
};

}  // namespace

// Peer-to-peer mode (embc_exchange_set_mode(ex, 1)): every rank's window,
// shared with its peers through CUDA IPC.  Layout of a receiver's window for
// one direction (every rank computes every window's layout from the call's
// shapes and codecs): data[R] | ack[R] flags (u64), then per source s its
// chunks' lengths and slot-relative offsets (u64, sources in rank order), then
// per source a slot holding its chunks (capacity = the chunks' encode bounds).
struct P2PState {
  size_t cap = 0;                 // window bytes (same on every rank)
  uint8_t* win = nullptr;         // this rank's window
  std::vector<uint8_t*> peer;     // every rank's window as mapped here (peer[rank] = win)
  uint64_t* d_epoch = nullptr;    // exchange counter, bumped on the device
  uint32_t* d_timeout = nullptr;  // a flag wait gave up
  void* d_sig = nullptr;          // device pointer arrays for the signal kernels (2 x R)
};

struct embc_exchange {
  int device = 0, rank = 0, R = 1;
  uint32_t groups = 1;
  int mode = 0;  // 0: NCCL metadata + payload rounds; 1: peer-to-peer windows
  P2PState p2p;
  ncclComm_t comm = nullptr;
  embc_ctx* enc = nullptr;
  embc_ctx* dec = nullptr;
  cudaStream_t s_enc = nullptr, s_comm = nullptr, s_dec = nullptr;
  cudaEvent_t ev_in = nullptr, ev_out = nullptr;
  std::vector<Group> g;
  embc_error last{};
};

namespace {

embc_status fail(embc_exchange* ex, embc_status st, int reason, const std::string& msg) {
  ex->last = embc_error{};
  ex->last.status = st;
  ex->last.reason = reason;
  std::snprintf(ex->last.message, sizeof(ex->last.message), "%s", msg.c_str());
  return st;
}

embc_status cuda_fail(embc_exchange* ex, cudaError_t e, const char* where) {
  return fail(ex, EMBC_ERR_CUDA, 0, std::string("CUDA error in exchange ") + where + ": " + cudaGetErrorString(e));
}

embc_status nccl_fail(embc_exchange* ex, ncclResult_t r, const char* where) {
  return fail(ex, EMBC_ERR_NCCL, 0,
              std::string("NCCL error in exchange ") + where + ": " + nccl().GetErrorString(r));
}

// A codec failure: the context's record, with the reference's rank/stage
// attribution (commsim.hpp:317-319, :398-401).
embc_status codec_fail(embc_exchange* ex, embc_ctx* ctx, embc_status st, const std::string& stage) {
  embc_error e{};
  embc_get_error(ctx, &e);
  ex->last = e;
  const std::string m = "rank " + std::to_string(ex->rank) + " " + stage + ": " + e.message;
  std::snprintf(ex->last.message, sizeof(ex->last.message), "%s", m.c_str());
  return st;
}

std::vector<uint32_t> owned(uint32_t T, int R, int r) {
  std::vector<uint32_t> v;
  for (uint32_t t = static_cast<uint32_t>(r); t < T; t += static_cast<uint32_t>(R)) v.push_back(t);
  return v;
}

// Positions of group k when n items are cut into G runs (every rank uses the
// same G so the rounds line up).
std::pair<size_t, size_t> split(size_t n, size_t G, size_t k) { return {k * n / G, (k + 1) * n / G}; }

// One direction of the exchange.  jobs[k] are group k's chunks in
// (destination, table) order; recv[k][src] the chunks src sends in its order.
embc_status run(embc_exchange* ex, uint32_t dim, uint32_t batch, const double* ebs, const uint8_t* codecs,
                uint32_t window, const std::vector<std::vector<SendJob>>& jobs,
                const std::vector<std::vector<std::vector<RecvChunk>>>& recv, embc_exchange_stats* stats,
                cudaStream_t stream, const char* dir) {
  const Nccl& N = nccl();
  const int R = ex->R;
  const size_t G = jobs.size();
  embc_exchange_stats st{};
  embc_status first = EMBC_OK;  // a data failure: reported after both rounds complete on every rank
  const uint64_t chunk_values = static_cast<uint64_t>(batch) * dim;
  cudaError_t ce = cudaEventRecord(ex->ev_in, stream);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(ex->s_enc, ex->ev_in, 0);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(ex->s_dec, ex->ev_in, 0);  // outputs may be in use on `stream`
  if (ce != cudaSuccess) return cuda_fail(ex, ce, "stream fork");
  // stage 1 for every group up front (compression of group k+1 overlaps the
  // transfer of group k)
  for (size_t k = 0; k < G; ++k) {
    Group& gr = ex->g[k];
    const auto& J = jobs[k];
    std::vector<embc_job> cj(J.size());
    for (size_t j = 0; j < J.size(); ++j) {
      embc_job& c = cj[j];
      std::memset(&c, 0, sizeof(c));
      c.src = J[j].src;
      c.dim = dim;
      c.n = batch;
      c.eb = ebs[J[j].table];
      c.window = window;
      c.codec = codecs[J[j].table];
      c.src_kind = EMBC_SRC_F32;
    }
    const uint64_t bound = embc_encode_bound(cj.data(), static_cast<uint32_t>(cj.size()), EMBC_LAYOUT_CHUNKS);
    if ((ce = gr.send.reserve(bound + 16)) != cudaSuccess || (ce = gr.lens.reserve(8 * J.size() + 8)) != cudaSuccess ||
        (ce = gr.meta.reserve(kMeta * J.size() + 8)) != cudaSuccess)
      return cuda_fail(ex, ce, "buffer allocation");
    // a job the encoder aborts on (non-finite value, ...) announces 0 bytes,
    // so every rank still completes both rounds; the failure surfaces below
    if ((ce = cudaMemsetAsync(gr.lens.p, 0, 8 * J.size() + 8, ex->s_enc)) != cudaSuccess ||
        (ce = cudaMemsetAsync(gr.meta.p, 0, kMeta * J.size() + 8, ex->s_enc)) != cudaSuccess)
      return cuda_fail(ex, ce, "buffer reset");
    if (!cj.empty()) {
      const embc_status s = embc_encode(ex->enc, cj.data(), static_cast<uint32_t>(cj.size()), EMBC_LAYOUT_CHUNKS,
                                        gr.send.as<uint8_t>(), gr.send.cap, nullptr, gr.lens.as<uint64_t>(),
                                        gr.meta.as<uint8_t>(), nullptr, ex->s_enc);
      // a host-known failure (invalid bound, ...): this rank announces empty
      // chunks and still takes part in both rounds
      if (s != EMBC_OK && first == EMBC_OK) first = codec_fail(ex, ex->enc, s, std::string(dir) + " compress stage");
    }
    if ((ce = cudaEventRecord(gr.encoded, ex->s_enc)) != cudaSuccess) return cuda_fail(ex, ce, "event");
  }
  for (size_t k = 0; k < G; ++k) {
    Group& gr = ex->g[k];
    const auto& J = jobs[k];
    std::vector<size_t> send_cnt(R, 0), recv_cnt(R, 0);
    for (const SendJob& j : J) ++send_cnt[j.dst];
    size_t nrecv = 0;
    for (int s = 0; s < R; ++s) nrecv += (recv_cnt[s] = recv[k][s].size());
    if ((ce = gr.meta_recv.reserve(kMeta * nrecv + 8)) != cudaSuccess ||
        (ce = gr.host.reserve(8 * J.size() + kMeta * nrecv + 8)) != cudaSuccess)
      return cuda_fail(ex, ce, "buffer allocation");
    if ((ce = cudaStreamWaitEvent(ex->s_comm, gr.encoded, 0)) != cudaSuccess) return cuda_fail(ex, ce, "stream wait");
    // stage 2: metadata round, 25 B per chunk (commsim.hpp:321-330)
    ncclResult_t nr = N.GroupStart();
    size_t so = 0, ro = 0;
    for (int p = 0; p < R && nr == ncclSuccess; ++p) {
      if (send_cnt[p]) nr = N.Send(gr.meta.as<uint8_t>() + kMeta * so, kMeta * send_cnt[p], ncclUint8, p, ex->comm, ex->s_comm);
      if (nr == ncclSuccess && recv_cnt[p])
        nr = N.Recv(gr.meta_recv.as<uint8_t>() + kMeta * ro, kMeta * recv_cnt[p], ncclUint8, p, ex->comm, ex->s_comm);
      so += send_cnt[p];
      ro += recv_cnt[p];
    }
    const ncclResult_t ne = N.GroupEnd();
    if (nr != ncclSuccess) return nccl_fail(ex, nr, "metadata round");
    if (ne != ncclSuccess) return nccl_fail(ex, ne, "metadata round");
    uint8_t* h = gr.host.as<uint8_t>();
    if (!J.empty() && (ce = cudaMemcpyAsync(h, gr.lens.p, 8 * J.size(), cudaMemcpyDeviceToHost, ex->s_comm)) != cudaSuccess)
      return cuda_fail(ex, ce, "length readback");
    if (nrecv && (ce = cudaMemcpyAsync(h + 8 * J.size(), gr.meta_recv.p, kMeta * nrecv, cudaMemcpyDeviceToHost,
                                       ex->s_comm)) != cudaSuccess)
      return cuda_fail(ex, ce, "metadata readback");
    // the host needs the byte counts: the one wait per group
    if ((ce = cudaStreamSynchronize(ex->s_comm)) != cudaSuccess) return cuda_fail(ex, ce, "metadata wait");
    std::vector<uint64_t> lens(J.size());
    std::memcpy(lens.data(), h, 8 * J.size());
    std::vector<uint64_t> send_bytes(R, 0), recv_bytes(R, 0);
    for (size_t j = 0; j < J.size(); ++j) {
      send_bytes[J[j].dst] += lens[j];
      st.sent_values += chunk_values;
      st.sent_bytes += lens[j];
      if (static_cast<int>(J[j].dst) != ex->rank) {
        st.payload_bytes += lens[j];
        st.metadata_bytes += kMeta;
        st.uncompressed_bytes += 4 * chunk_values;
      }
    }
    // parse_metadata (container.hpp:211-221) of what arrives; the decode plan
    std::vector<embc_chunk_ref> refs;
    refs.reserve(nrecv);
    uint64_t off = 0;
    size_t m = 0;
    for (int s = 0; s < R; ++s) {
      for (const RecvChunk& rc : recv[k][s]) {
        const uint8_t* rec = h + 8 * J.size() + kMeta * m++;
        uint64_t clen;
        uint32_t mdim, mcount;
        std::memcpy(&clen, rec, 8);
        std::memcpy(&mdim, rec + 17, 4);
        std::memcpy(&mcount, rec + 21, 4);
        if (mdim != dim || mcount != batch) {  // commsim.hpp:371-376; the bytes still arrive
          if (first == EMBC_OK)
            first = fail(ex, EMBC_ERR_FORMAT, EMBC_R_META_MISMATCH,
                         "rank " + std::to_string(ex->rank) + " decompress stage (from rank " + std::to_string(s) +
                             "): metadata from rank " + std::to_string(s) + " disagrees with its chunk");
          off += clen;
          recv_bytes[s] += clen;
          continue;
        }
        embc_chunk_ref r{};
        r.offset = off;
        r.length = clen;
        r.out = rc.out;
        r.dim = dim;
        r.count = batch;
        r.codec = rec[8];
        refs.push_back(r);
        off += clen;
        recv_bytes[s] += clen;
        st.recv_values += chunk_values;
        st.recv_bytes += clen;
      }
    }
    if ((ce = gr.recv.reserve(off + 16)) != cudaSuccess) return cuda_fail(ex, ce, "buffer allocation");
    // stage 3: payload round
    nr = N.GroupStart();
    uint64_t sofs = 0, rofs = 0;
    for (int p = 0; p < R && nr == ncclSuccess; ++p) {
      if (send_bytes[p]) nr = N.Send(gr.send.as<uint8_t>() + sofs, send_bytes[p], ncclUint8, p, ex->comm, ex->s_comm);
      if (nr == ncclSuccess && recv_bytes[p])
        nr = N.Recv(gr.recv.as<uint8_t>() + rofs, recv_bytes[p], ncclUint8, p, ex->comm, ex->s_comm);
      sofs += send_bytes[p];
      rofs += recv_bytes[p];
    }
    const ncclResult_t ne2 = N.GroupEnd();
    if (nr != ncclSuccess) return nccl_fail(ex, nr, "payload round");
    if (ne2 != ncclSuccess) return nccl_fail(ex, ne2, "payload round");
    if ((ce = cudaEventRecord(gr.arrived, ex->s_comm)) != cudaSuccess ||
        (ce = cudaStreamWaitEvent(ex->s_dec, gr.arrived, 0)) != cudaSuccess)
      return cuda_fail(ex, ce, "stream join");
    // stage 4: decode into the caller's tensors (headers checked on the device)
    if (!refs.empty()) {
      const embc_status s = embc_decode(ex->dec, gr.recv.as<uint8_t>(), refs.data(), static_cast<uint32_t>(refs.size()),
                                        EMBC_OUT_F32, 0, ex->s_dec);
      if (s != EMBC_OK && first == EMBC_OK) first = codec_fail(ex, ex->dec, s, std::string(dir) + " decompress stage");
    }
  }
  if ((ce = cudaEventRecord(ex->ev_out, ex->s_dec)) != cudaSuccess ||
      (ce = cudaStreamWaitEvent(stream, ex->ev_out, 0)) != cudaSuccess)
    return cuda_fail(ex, ce, "stream join");
  // device-recorded codec failures (non-finite values, malformed chunks) surface
  // here, the compress stage's first (commsim.hpp:317-319, :398-401)
  // both contexts are synchronised (and their records cleared) before either
  // failure is reported, so the next call starts clean
  const embc_status se = embc_sync(ex->enc, ex->s_enc);
  const embc_status sd = embc_sync(ex->dec, ex->s_dec);
  if (se != EMBC_OK) return codec_fail(ex, ex->enc, se, std::string(dir) + " compress stage");
  if (first != EMBC_OK) return first;
  if (sd != EMBC_OK) return codec_fail(ex, ex->dec, sd, std::string(dir) + " decompress stage");
  if (stats) *stats = st;
  return EMBC_OK;
}

size_t group_count(const embc_exchange* ex, uint32_t T) {
  size_t mx = 0;
  for (int r = 0; r < ex->R; ++r) mx = std::max(mx, owned(T, ex->R, r).size());
  return std::max<size_t>(1, std::min<size_t>(ex->groups, std::max<size_t>(mx, 1)));
}

embc_status prepare_groups(embc_exchange* ex, size_t G) {
  while (ex->g.size() < G) {
    ex->g.emplace_back();
    Group& gr = ex->g.back();
    cudaError_t ce = cudaEventCreateWithFlags(&gr.encoded, cudaEventDisableTiming);
    if (ce == cudaSuccess) ce = cudaEventCreateWithFlags(&gr.arrived, cudaEventDisableTiming);
    if (ce != cudaSuccess) return cuda_fail(ex, ce, "event creation");
  }
  return EMBC_OK;
}

bool bad_args(embc_exchange* ex, uint32_t T, uint32_t dim, uint32_t batch, const void* a, const void* b,
              const void* c, const void* d) {
  return !ex || !T || !dim || !batch || !a || !b || !c || !d;
}

// ---- peer-to-peer mode ---------------------------------------------------------

// Upper bound on one chunk's serialized bytes (embc_encode_bound of the job).
uint64_t chunk_cap(uint32_t dim, uint32_t batch, uint8_t codec) {
  embc_job j{};
  j.dim = dim;
  j.n = batch;
  j.eb = 1.0;
  j.window = 255;
  j.codec = codec;
  return embc_encode_bound(&j, 1, EMBC_LAYOUT_CHUNKS);
}

// A receiver's window for one direction: tables_of(s, r) lists the tables s
// sends to r, in s's job order.
struct Layout {
  std::vector<uint32_t> nin;     // chunks per source
  std::vector<uint64_t> pre;     // index of source s's first chunk
  std::vector<std::vector<uint64_t>> caps;
  std::vector<uint64_t> slot;    // byte offset of source s's slot
  std::vector<uint64_t> slot_cap;
  uint64_t off_lens = 0, off_offs = 0, total = 0;
};

Layout layout_of(int R, int r, uint32_t dim, uint32_t batch, const uint8_t* codecs,
                 const std::function<std::vector<uint32_t>(int, int)>& tables_of) {
  Layout L;
  L.nin.resize(R);
  L.pre.resize(R);
  L.caps.resize(R);
  L.slot.resize(R);
  L.slot_cap.resize(R);
  uint64_t n = 0;
  for (int s = 0; s < R; ++s) {
    const auto t = tables_of(s, r);
    L.nin[s] = static_cast<uint32_t>(t.size());
    L.pre[s] = n;
    n += t.size();
    uint64_t c = 0;
    for (uint32_t x : t) {
      L.caps[s].push_back(chunk_cap(dim, batch, codecs[x]));
      c += L.caps[s].back();
    }
    L.slot_cap[s] = c;
  }
  L.off_lens = 16ull * R;
  L.off_offs = L.off_lens + 8 * n;
  uint64_t o = (L.off_offs + 8 * n + 255) & ~255ull;
  for (int s = 0; s < R; ++s) {
    L.slot[s] = o;
    o = (o + L.slot_cap[s] + 255) & ~255ull;
  }
  L.total = o;
  return L;
}

// A grouped send/recv of `bytes` from every rank to every rank (setup only).
embc_status all_to_all_bytes(embc_exchange* ex, const void* d_send, void* d_recv, size_t bytes) {
  const Nccl& N = nccl();
  ncclResult_t nr = N.GroupStart();
  for (int p = 0; p < ex->R && nr == ncclSuccess; ++p) {
    nr = N.Send(static_cast<const uint8_t*>(d_send), bytes, ncclUint8, p, ex->comm, ex->s_comm);
    if (nr == ncclSuccess) nr = N.Recv(static_cast<uint8_t*>(d_recv) + bytes * p, bytes, ncclUint8, p, ex->comm, ex->s_comm);
  }
  const ncclResult_t ne = N.GroupEnd();
  if (nr != ncclSuccess) return nccl_fail(ex, nr, "window setup");
  if (ne != ncclSuccess) return nccl_fail(ex, ne, "window setup");
  const cudaError_t ce = cudaStreamSynchronize(ex->s_comm);
  return ce == cudaSuccess ? EMBC_OK : cuda_fail(ex, ce, "window setup");
}

void p2p_release(embc_exchange* ex) {
  P2PState& P = ex->p2p;
  for (int r = 0; r < static_cast<int>(P.peer.size()); ++r)
    if (r != ex->rank && P.peer[r]) cudaIpcCloseMemHandle(P.peer[r]);
  P.peer.clear();
  if (P.win) cudaFree(P.win);
  P.win = nullptr;
  P.cap = 0;
}

// Every rank's window of at least `need` bytes (collective: every rank makes
// the same calls, so all grow together), mapped on every peer.
embc_status p2p_window(embc_exchange* ex, uint64_t need) {
  P2PState& P = ex->p2p;
  cudaError_t ce;
  if (!P.d_epoch) {
    void* p = nullptr;
    if ((ce = cudaMalloc(&p, 16)) != cudaSuccess) return cuda_fail(ex, ce, "window setup");
    cudaMemset(p, 0, 16);
    P.d_epoch = static_cast<uint64_t*>(p);
    P.d_timeout = reinterpret_cast<uint32_t*>(static_cast<uint8_t*>(p) + 8);
    if ((ce = cudaMalloc(&P.d_sig, sizeof(void*) * 2 * ex->R)) != cudaSuccess) return cuda_fail(ex, ce, "window setup");
  }
  if (need <= P.cap) return EMBC_OK;
  // peers may still read the old windows: drain every stream, then a round trip
  cudaDeviceSynchronize();
  DevBuf tok;
  if ((ce = tok.reserve(16ull * ex->R)) != cudaSuccess) return cuda_fail(ex, ce, "window setup");
  embc_status st = all_to_all_bytes(ex, tok.p, tok.as<uint8_t>() + 8ull * ex->R, 8);
  if (st != EMBC_OK) return st;
  p2p_release(ex);
  const uint64_t cap = std::max<uint64_t>(need + need / 4, 1 << 20);
  if ((ce = cudaMalloc(&P.win, cap)) != cudaSuccess) return cuda_fail(ex, ce, "window allocation");
  // flags start at 0 (epoch 0 never signalled), so a fresh window waits correctly
  if ((ce = cudaMemset(P.win, 0, 16ull * ex->R)) != cudaSuccess) return cuda_fail(ex, ce, "window setup");
  P.cap = cap;
  P.peer.assign(ex->R, nullptr);
  P.peer[ex->rank] = P.win;
  if (ex->R > 1) {
    cudaIpcMemHandle_t h;
    if ((ce = cudaIpcGetMemHandle(&h, P.win)) != cudaSuccess) return cuda_fail(ex, ce, "window handle");
    DevBuf hb;
    if ((ce = hb.reserve(sizeof(h) * (ex->R + 1))) != cudaSuccess) return cuda_fail(ex, ce, "window setup");
    cudaMemcpy(hb.p, &h, sizeof(h), cudaMemcpyHostToDevice);
    st = all_to_all_bytes(ex, hb.p, hb.as<uint8_t>() + sizeof(h), sizeof(h));
    if (st != EMBC_OK) return st;
    std::vector<cudaIpcMemHandle_t> all(ex->R);
    cudaMemcpy(all.data(), hb.as<uint8_t>() + sizeof(h), sizeof(h) * ex->R, cudaMemcpyDeviceToHost);
    for (int r = 0; r < ex->R; ++r) {
      if (r == ex->rank) continue;
      void* p = nullptr;
      if ((ce = cudaIpcOpenMemHandle(&p, all[r], cudaIpcMemLazyEnablePeerAccess)) != cudaSuccess)
        return cuda_fail(ex, ce, "peer window mapping");
      P.peer[r] = static_cast<uint8_t*>(p);
    }
  }
  // pointer tables of the signal kernels: data[me] in every destination's
  // window, ack[me] in every source's window
  std::vector<uint64_t*> sig(2 * ex->R);
  for (int r = 0; r < ex->R; ++r) {
    sig[r] = reinterpret_cast<uint64_t*>(P.peer[r]) + ex->rank;
    sig[ex->R + r] = reinterpret_cast<uint64_t*>(P.peer[r]) + ex->R + ex->rank;
  }
  cudaMemcpy(P.d_sig, sig.data(), sizeof(void*) * sig.size(), cudaMemcpyHostToDevice);
  // every rank mapped every window before anyone writes into one
  return all_to_all_bytes(ex, tok.p, tok.as<uint8_t>() + 8ull * ex->R, 8);
}

// One direction over the windows: this rank's chunks for destination d go
// straight into d's window (its own encode kernels store over NVLink), then
// a flag per destination; the receive side waits for every source's flag and
// decodes from its own window with the device-planned decoder (lengths never
// visit the host), then acknowledges.  No host synchronisation unless
// `stats` is requested.
embc_status run_p2p(embc_exchange* ex, uint32_t T, uint32_t dim, uint32_t batch, const double* ebs,
                    const uint8_t* codecs, uint32_t window,
                    const std::function<std::vector<uint32_t>(int, int)>& tables_of,
                    const std::function<const float*(uint32_t, int)>& src_of,
                    const std::function<float*(uint32_t, int)>& out_of, embc_exchange_stats* stats,
                    cudaStream_t stream, const char* dir) {
  const int R = ex->R, me = ex->rank;
  std::vector<Layout> L(R);
  uint64_t need = 0;
  for (int r = 0; r < R; ++r) {
    L[r] = layout_of(R, r, dim, batch, codecs, tables_of);
    need = std::max(need, L[r].total);
  }
  (void)T;
  embc_status st = p2p_window(ex, need);
  if (st != EMBC_OK) return st;
  P2PState& P = ex->p2p;
  auto* sig = static_cast<uint64_t* const*>(P.d_sig);
  cudaError_t ce = embc_p2p::bump(P.d_epoch, stream);
  if (ce == cudaSuccess) ce = cudaEventRecord(ex->ev_in, stream);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(ex->s_enc, ex->ev_in, 0);
  if (ce == cudaSuccess) ce = cudaStreamWaitEvent(ex->s_dec, ex->ev_in, 0);
  // send side: every destination has decoded what this rank wrote last time
  if (ce == cudaSuccess)
    ce = embc_p2p::wait(reinterpret_cast<const uint64_t*>(P.win) + R, R, P.d_epoch, 1, P.d_timeout, ex->s_enc);
  if (ce != cudaSuccess) return cuda_fail(ex, ce, "p2p send setup");
  embc_status first = EMBC_OK;
  embc_exchange_stats stt{};
  const uint64_t chunk_values = static_cast<uint64_t>(batch) * dim;
  for (int d = 0; d < R; ++d) {
    const auto tabs = tables_of(me, d);
    if (tabs.empty()) continue;
    const Layout& Ld = L[d];
    std::vector<embc_job> cj(tabs.size());
    for (size_t j = 0; j < tabs.size(); ++j) {
      embc_job& c = cj[j];
      std::memset(&c, 0, sizeof(c));
      c.src = src_of(tabs[j], d);
      c.dim = dim;
      c.n = batch;
      c.eb = ebs[tabs[j]];
      c.window = window;
      c.codec = codecs[tabs[j]];
      c.src_kind = EMBC_SRC_F32;
    }
    uint8_t* w = P.peer[d];
    uint64_t* lens = reinterpret_cast<uint64_t*>(w + Ld.off_lens) + Ld.pre[me];
    uint64_t* offs = reinterpret_cast<uint64_t*>(w + Ld.off_offs) + Ld.pre[me];
    const embc_status s = embc_encode(ex->enc, cj.data(), static_cast<uint32_t>(cj.size()), EMBC_LAYOUT_CHUNKS,
                                      w + Ld.slot[me], Ld.slot_cap[me], offs, lens, nullptr, nullptr, ex->s_enc);
    if (s != EMBC_OK && first == EMBC_OK) first = codec_fail(ex, ex->enc, s, std::string(dir) + " compress stage");
  }
  if ((ce = embc_p2p::signal(sig, R, P.d_epoch, ex->s_enc)) != cudaSuccess) return cuda_fail(ex, ce, "p2p signal");
  Group& gr = ex->g[0];
  if ((ce = cudaEventRecord(gr.encoded, ex->s_enc)) != cudaSuccess) return cuda_fail(ex, ce, "event");
  // receive side: this rank's own slot comes from its encode stream (an event
  // dependency, so no wait relies on concurrent kernels); peers' by their flags
  if ((ce = cudaStreamWaitEvent(ex->s_dec, gr.encoded, 0)) != cudaSuccess ||
      (ce = embc_p2p::wait(reinterpret_cast<const uint64_t*>(P.win), R, P.d_epoch, 0, P.d_timeout, ex->s_dec)) !=
          cudaSuccess)
    return cuda_fail(ex, ce, "p2p receive setup");
  const Layout& Lm = L[me];
  std::vector<embc_chunk_ref> refs;
  for (int s = 0; s < R; ++s) {
    const auto tabs = tables_of(s, me);
    for (size_t k = 0; k < tabs.size(); ++k) {
      embc_chunk_ref r{};
      r.offset = Lm.slot[s];
      r.length = Lm.caps[s][k];
      r.out = out_of(tabs[k], s);
      r.dim = dim;
      r.count = batch;
      r.codec = codecs[tabs[k]];
      refs.push_back(r);
    }
  }
  if (!refs.empty()) {
    const embc_status s = embc_decode_dev(ex->dec, P.win, refs.data(), static_cast<uint32_t>(refs.size()),
                                          reinterpret_cast<const uint64_t*>(P.win + Lm.off_offs),
                                          reinterpret_cast<const uint64_t*>(P.win + Lm.off_lens), EMBC_OUT_F32, 0,
                                          ex->s_dec);
    if (s != EMBC_OK && first == EMBC_OK) first = codec_fail(ex, ex->dec, s, std::string(dir) + " decompress stage");
  }
  if ((ce = embc_p2p::signal(sig + R, R, P.d_epoch, ex->s_dec)) != cudaSuccess) return cuda_fail(ex, ce, "p2p ack");
  if ((ce = cudaEventRecord(ex->ev_out, ex->s_dec)) != cudaSuccess ||
      (ce = cudaStreamWaitEvent(stream, ex->ev_out, 0)) != cudaSuccess ||
      (ce = cudaStreamWaitEvent(stream, gr.encoded, 0)) != cudaSuccess)
    return cuda_fail(ex, ce, "stream join");
  if (first != EMBC_OK) return first;
  if (!stats) return EMBC_OK;  // asynchronous (and graph-capturable): failures at embc_exchange_sync
  // accounting (commsim.hpp:322-353): this rank's chunk lengths as its peers received them
  st = embc_exchange_sync(ex);
  if (st != EMBC_OK) return st;
  for (int d = 0; d < R; ++d) {
    const uint32_t n = L[d].nin[me];
    if (!n) continue;
    std::vector<uint64_t> lens(n);
    cudaMemcpy(lens.data(), reinterpret_cast<uint64_t*>(P.peer[d] + L[d].off_lens) + L[d].pre[me], 8 * n,
               cudaMemcpyDeviceToHost);
    for (uint64_t l : lens) {
      stt.sent_values += chunk_values;
      stt.sent_bytes += l;
      if (d != me) {
        stt.payload_bytes += l;
        stt.metadata_bytes += kMeta;
        stt.uncompressed_bytes += 4 * chunk_values;
      }
    }
  }
  {
    std::vector<uint64_t> lens(refs.size());
    if (!refs.empty())
      cudaMemcpy(lens.data(), P.win + Lm.off_lens, 8 * refs.size(), cudaMemcpyDeviceToHost);
    for (uint64_t l : lens) {
      stt.recv_values += chunk_values;
      stt.recv_bytes += l;
    }
  }
  *stats = stt;
  return EMBC_OK;
}

}  // namespace

extern "C" {

embc_status embc_exchange_unique_id(uint8_t out[128]) {
  const Nccl& N = nccl();
  if (!out) return EMBC_ERR_ARGUMENT;
  if (!N.ok) return EMBC_ERR_UNSUPPORTED;
  ncclUniqueId id;
  if (N.GetUniqueId(&id) != ncclSuccess) return EMBC_ERR_NCCL;
  std::memcpy(out, id.internal, NCCL_UNIQUE_ID_BYTES);
  return EMBC_OK;
}

embc_status embc_exchange_create(int device, int rank, int nranks, const uint8_t id[128], uint32_t groups,
                                 embc_exchange** out) {
  if (!out || !id || nranks < 1 || rank < 0 || rank >= nranks) return EMBC_ERR_ARGUMENT;
  *out = nullptr;
  const Nccl& N = nccl();
  if (!N.ok) return EMBC_ERR_UNSUPPORTED;
  if (cudaSetDevice(device) != cudaSuccess) return EMBC_ERR_CUDA;
  auto* ex = new embc_exchange;
  ex->device = device;
  ex->rank = rank;
  ex->R = nranks;
  ex->groups = std::max<uint32_t>(groups, 1);
  ncclUniqueId uid;
  std::memcpy(uid.internal, id, NCCL_UNIQUE_ID_BYTES);
  if (N.CommInitRank(&ex->comm, nranks, uid, rank) != ncclSuccess) {
    delete ex;
    return EMBC_ERR_NCCL;
  }
  embc_status st = embc_ctx_create(device, &ex->enc);
  if (st == EMBC_OK) st = embc_ctx_create(device, &ex->dec);
  cudaError_t ce = cudaSuccess;
  if (st == EMBC_OK) ce = cudaStreamCreateWithFlags(&ex->s_enc, cudaStreamNonBlocking);
  if (st == EMBC_OK && ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&ex->s_comm, cudaStreamNonBlocking);
  if (st == EMBC_OK && ce == cudaSuccess) ce = cudaStreamCreateWithFlags(&ex->s_dec, cudaStreamNonBlocking);
  if (st == EMBC_OK && ce == cudaSuccess) ce = cudaEventCreateWithFlags(&ex->ev_in, cudaEventDisableTiming);
  if (st == EMBC_OK && ce == cudaSuccess) ce = cudaEventCreateWithFlags(&ex->ev_out, cudaEventDisableTiming);
  if (st != EMBC_OK || ce != cudaSuccess) {
    embc_exchange_destroy(ex);
    return st != EMBC_OK ? st : EMBC_ERR_CUDA;
  }
  *out = ex;
  return EMBC_OK;
}

void embc_exchange_destroy(embc_exchange* ex) {
  if (!ex) return;
  cudaSetDevice(ex->device);
  if (ex->s_enc) cudaStreamSynchronize(ex->s_enc);
  if (ex->s_comm) cudaStreamSynchronize(ex->s_comm);
  if (ex->s_dec) cudaStreamSynchronize(ex->s_dec);
  for (Group& gr : ex->g) {
    if (gr.encoded) cudaEventDestroy(gr.encoded);
    if (gr.arrived) cudaEventDestroy(gr.arrived);
  }
  ex->g.clear();
  p2p_release(ex);
  if (ex->p2p.d_epoch) cudaFree(ex->p2p.d_epoch);
  if (ex->p2p.d_sig) cudaFree(ex->p2p.d_sig);
  if (ex->comm) nccl().CommDestroy(ex->comm);
  if (ex->enc) embc_ctx_destroy(ex->enc);
  if (ex->dec) embc_ctx_destroy(ex->dec);
  for (cudaStream_t s : {ex->s_enc, ex->s_comm, ex->s_dec})
    if (s) cudaStreamDestroy(s);
  for (cudaEvent_t e : {ex->ev_in, ex->ev_out})
    if (e) cudaEventDestroy(e);
  delete ex;
}

embc_status embc_exchange_get_error(const embc_exchange* ex, embc_error* out) {
  if (!ex || !out) return EMBC_ERR_ARGUMENT;
  *out = ex->last;
  return EMBC_OK;
}

embc_status embc_exchange_fwd(embc_exchange* ex, uint32_t T, uint32_t dim, uint32_t batch,
                              const float* const* d_lookups, const double* ebs, const uint8_t* codecs,
                              uint32_t window, float* const* d_outs, embc_exchange_stats* stats, void* stream) {
  if (bad_args(ex, T, dim, batch, d_lookups, ebs, codecs, d_outs))
    return ex ? fail(ex, EMBC_ERR_ARGUMENT, 0, "invalid embc_exchange_fwd arguments") : EMBC_ERR_ARGUMENT;
  const int R = ex->R;
  const size_t G = group_count(ex, T);
  embc_status st = prepare_groups(ex, G);
  if (st != EMBC_OK) return st;
  const auto own = owned(T, R, ex->rank);
  const uint64_t rows = static_cast<uint64_t>(batch) * dim;
  if (ex->mode == 1) {
    cudaSetDevice(ex->device);
    return run_p2p(
        ex, T, dim, batch, ebs, codecs, window, [&](int s, int) { return owned(T, R, s); },
        [&](uint32_t t, int d) { return d_lookups[t] + d * rows; }, [&](uint32_t t, int) { return d_outs[t]; },
        stats, static_cast<cudaStream_t>(stream), "forward");
  }
  std::vector<std::vector<SendJob>> jobs(G);
  std::vector<std::vector<std::vector<RecvChunk>>> recv(G, std::vector<std::vector<RecvChunk>>(R));
  for (size_t k = 0; k < G; ++k) {
    const auto [a, b] = split(own.size(), G, k);
    for (int d = 0; d < R; ++d)
      for (size_t i = a; i < b; ++i)
        jobs[k].push_back(SendJob{own[i], static_cast<uint32_t>(d), d_lookups[own[i]] + d * rows});
    for (int s = 0; s < R; ++s) {
      const auto theirs = owned(T, R, s);
      const auto [c, e] = split(theirs.size(), G, k);
      for (size_t i = c; i < e; ++i) recv[k][s].push_back(RecvChunk{theirs[i], static_cast<uint32_t>(s), d_outs[theirs[i]]});
    }
  }
  cudaSetDevice(ex->device);
  return run(ex, dim, batch, ebs, codecs, window, jobs, recv, stats, static_cast<cudaStream_t>(stream), "forward");
}

embc_status embc_exchange_bwd(embc_exchange* ex, uint32_t T, uint32_t dim, uint32_t batch,
                              const float* const* d_grads, const double* ebs, const uint8_t* codecs,
                              uint32_t window, float* const* d_outs, embc_exchange_stats* stats, void* stream) {
  if (bad_args(ex, T, dim, batch, d_grads, ebs, codecs, d_outs))
    return ex ? fail(ex, EMBC_ERR_ARGUMENT, 0, "invalid embc_exchange_bwd arguments") : EMBC_ERR_ARGUMENT;
  const int R = ex->R;
  const size_t G = group_count(ex, T);
  embc_status st = prepare_groups(ex, G);
  if (st != EMBC_OK) return st;
  const auto own = owned(T, R, ex->rank);
  const uint64_t rows = static_cast<uint64_t>(batch) * dim;
  if (ex->mode == 1) {
    cudaSetDevice(ex->device);
    return run_p2p(
        ex, T, dim, batch, ebs, codecs, window, [&](int, int r) { return owned(T, R, r); },
        [&](uint32_t t, int) { return d_grads[t]; }, [&](uint32_t t, int s) { return d_outs[t] + s * rows; }, stats,
        static_cast<cudaStream_t>(stream), "backward");
  }
  std::vector<std::vector<SendJob>> jobs(G);
  std::vector<std::vector<std::vector<RecvChunk>>> recv(G, std::vector<std::vector<RecvChunk>>(R));
  for (size_t k = 0; k < G; ++k) {
    for (int d = 0; d < R; ++d) {
      const auto theirs = owned(T, R, d);
      const auto [a, b] = split(theirs.size(), G, k);
      for (size_t i = a; i < b; ++i) jobs[k].push_back(SendJob{theirs[i], static_cast<uint32_t>(d), d_grads[theirs[i]]});
    }
    const auto [c, e] = split(own.size(), G, k);
    for (int s = 0; s < R; ++s)
      for (size_t i = c; i < e; ++i)
        recv[k][s].push_back(RecvChunk{own[i], static_cast<uint32_t>(s), d_outs[own[i]] + s * rows});
  }
  cudaSetDevice(ex->device);
  return run(ex, dim, batch, ebs, codecs, window, jobs, recv, stats, static_cast<cudaStream_t>(stream), "backward");
}

// Raw fp32 exchange of the same tensors: one grouped send/recv, no metadata round.
static embc_status baseline(embc_exchange* ex, const std::vector<std::vector<const float*>>& to,
                            const std::vector<std::vector<float*>>& from, uint64_t chunk_values, cudaStream_t stream) {
  const Nccl& N = nccl();
  cudaSetDevice(ex->device);
  ncclResult_t nr = N.GroupStart();
  for (int p = 0; p < ex->R && nr == ncclSuccess; ++p) {
    for (const float* s : to[p])
      if (nr == ncclSuccess) nr = N.Send(s, chunk_values, ncclFloat32, p, ex->comm, stream);
    for (float* d : from[p])
      if (nr == ncclSuccess) nr = N.Recv(d, chunk_values, ncclFloat32, p, ex->comm, stream);
  }
  const ncclResult_t ne = N.GroupEnd();
  if (nr != ncclSuccess) return nccl_fail(ex, nr, "baseline");
  if (ne != ncclSuccess) return nccl_fail(ex, ne, "baseline");
  return EMBC_OK;
}

embc_status embc_exchange_baseline_fwd(embc_exchange* ex, uint32_t T, uint32_t dim, uint32_t batch,
                                       const float* const* d_lookups, float* const* d_outs, void* stream) {
  if (bad_args(ex, T, dim, batch, d_lookups, d_outs, d_outs, d_outs))
    return ex ? fail(ex, EMBC_ERR_ARGUMENT, 0, "invalid embc_exchange_baseline_fwd arguments") : EMBC_ERR_ARGUMENT;
  const uint64_t rows = static_cast<uint64_t>(batch) * dim;
  std::vector<std::vector<const float*>> to(ex->R);
  std::vector<std::vector<float*>> from(ex->R);
  for (int p = 0; p < ex->R; ++p) {
    for (uint32_t t : owned(T, ex->R, ex->rank)) to[p].push_back(d_lookups[t] + p * rows);
    for (uint32_t t : owned(T, ex->R, p)) from[p].push_back(d_outs[t]);
  }
  return baseline(ex, to, from, rows, static_cast<cudaStream_t>(stream));
}

embc_status embc_exchange_baseline_bwd(embc_exchange* ex, uint32_t T, uint32_t dim, uint32_t batch,
                                       const float* const* d_grads, float* const* d_outs, void* stream) {
  if (bad_args(ex, T, dim, batch, d_grads, d_outs, d_outs, d_outs))
    return ex ? fail(ex, EMBC_ERR_ARGUMENT, 0, "invalid embc_exchange_baseline_bwd arguments") : EMBC_ERR_ARGUMENT;
  const uint64_t rows = static_cast<uint64_t>(batch) * dim;
  std::vector<std::vector<const float*>> to(ex->R);
  std::vector<std::vector<float*>> from(ex->R);
  for (int p = 0; p < ex->R; ++p) {
    for (uint32_t t : owned(T, ex->R, p)) to[p].push_back(d_grads[t]);
    for (uint32_t t : owned(T, ex->R, ex->rank)) from[p].push_back(d_outs[t] + p * rows);
  }
  return baseline(ex, to, from, rows, static_cast<cudaStream_t>(stream));
}

embc_status embc_exchange_set_mode(embc_exchange* ex, int mode) {
  if (!ex || mode < 0 || mode > 1) return EMBC_ERR_ARGUMENT;
  ex->mode = mode;
  return EMBC_OK;
}

embc_status embc_exchange_reserve_capture(embc_exchange* ex, uint64_t bytes) {
  if (!ex) return EMBC_ERR_ARGUMENT;
  const embc_status a = embc_reserve_capture(ex->enc, bytes);
  return a != EMBC_OK ? a : embc_reserve_capture(ex->dec, bytes);
}

embc_status embc_exchange_sync(embc_exchange* ex) {
  if (!ex) return EMBC_ERR_ARGUMENT;
  cudaSetDevice(ex->device);
  const embc_status se = embc_sync(ex->enc, ex->s_enc);
  const embc_status sd = embc_sync(ex->dec, ex->s_dec);
  if (ex->p2p.d_timeout) {
    uint32_t t = 0;
    cudaMemcpy(&t, ex->p2p.d_timeout, 4, cudaMemcpyDeviceToHost);
    if (t) {
      cudaMemset(ex->p2p.d_timeout, 0, 4);
      return fail(ex, EMBC_ERR_NCCL, 0, "rank " + std::to_string(ex->rank) + ": a peer did not signal its window");
    }
  }
  if (se != EMBC_OK) return codec_fail(ex, ex->enc, se, "compress stage");
  if (sd != EMBC_OK) return codec_fail(ex, ex->dec, sd, "decompress stage");
  return EMBC_OK;
}

embc_status embc_exchange_timing_enable(embc_exchange* ex, int on) {
  if (!ex) return EMBC_ERR_ARGUMENT;
  embc_timing_enable(ex->enc, on);
  return embc_timing_enable(ex->dec, on);
}

int embc_exchange_timing_collect(embc_exchange* ex, char* names, size_t names_cap, float* ms, int max_entries) {
  if (!ex) return -1;
  const int a = embc_timing_collect(ex->enc, ex->s_enc, names, names_cap, ms, max_entries);
  if (a < 0) return a;
  size_t used = 0;
  for (int i = 0; i < a; ++i) used += std::strlen(names + used) + 1;
  const int b = embc_timing_collect(ex->dec, ex->s_dec, names + used, names_cap - used, ms + a, max_entries - a);
  return b < 0 ? b : a + b;
}

// ---- unpack (container.hpp:258-292): the offset-table validation ------------
embc_status embc_unpack(const uint8_t* buf, uint64_t len, uint64_t* offs, uint64_t* lens, uint32_t cap,
                        uint32_t* count, embc_error* err) {
  auto fmt = [&](int reason, uint64_t index, uint64_t a, uint64_t b, const std::string& msg) {
    if (err) {
      *err = embc_error{};
      err->status = EMBC_ERR_FORMAT;
      err->reason = reason;
      err->index = index;
      err->a = a;
      err->b = b;
      std::snprintf(err->message, sizeof(err->message), "%s", msg.c_str());
    }
    return EMBC_ERR_FORMAT;
  };
  auto need = [&](uint64_t pos, uint64_t n) -> bool { return len - pos >= n && pos <= len; };
  if (!count || (!buf && len)) return EMBC_ERR_ARGUMENT;
  uint64_t pos = 0;
  if (!need(pos, 4))  // ByteReader::need (bytes.hpp:157-162)
    return fmt(EMBC_R_TRUNCATED, 0, 4, len, "truncated input: need 4 bytes at offset 0, have " + std::to_string(len));
  uint32_t R;
  std::memcpy(&R, buf, 4);
  pos = 4;
  std::vector<std::pair<uint64_t, uint64_t>> table;
  table.reserve(std::min<uint64_t>(R, len / 16 + 1));
  for (uint32_t i = 0; i < R; ++i) {
    uint64_t v[2];
    for (int k = 0; k < 2; ++k) {
      if (!need(pos, 8))
        return fmt(EMBC_R_TRUNCATED, pos, 8, len - pos,
                   "truncated input: need 8 bytes at offset " + std::to_string(pos) + ", have " +
                       std::to_string(len - pos));
      std::memcpy(&v[k], buf + pos, 8);
      pos += 8;
    }
    table.emplace_back(v[0], v[1]);
  }
  uint64_t expected = 4 + 16ull * R;
  for (uint32_t i = 0; i < R; ++i) {
    const auto [o, l] = table[i];
    if (o != expected)
      return fmt(EMBC_R_PACK_OFFSET, i, o, expected,
                 "send buffer offset " + std::to_string(o) + " for entry " + std::to_string(i) +
                     " overlaps or skips bytes (expected " + std::to_string(expected) + ")");
    if (o + l > len) return fmt(EMBC_R_PACK_OVERRUN, i, 0, 0, "send buffer entry " + std::to_string(i) + " runs past the end");
    expected = o + l;
  }
  if (expected != len)
    return fmt(EMBC_R_PACK_TRAILING, 0, len - expected, 0,
               "send buffer has " + std::to_string(len - expected) + " unclaimed trailing bytes");
  *count = R;
  for (uint32_t i = 0; i < R && i < cap; ++i) {
    if (offs) offs[i] = table[i].first;
    if (lens) lens[i] = table[i].second;
  }
  return EMBC_OK;
}

}  // extern "C"
