// hb_runtime.cu -- error state, launch accounting, NCCL plumbing and the
// per-rank iteration engine (the schedule of driver.py:110-149, run on one
// CUDA stream, optionally as a replayed CUDA graph of one iteration).

#include <dlfcn.h>
#include <stdarg.h>
#include <stddef.h>
#include <stdio.h>
#include <string.h>

#include <atomic>
#include <vector>

#include "hb_common.cuh"

// NCCL's header from the venv (2.28.x) for the types; the functions are
// resolved with dlsym on first use, so single-GPU use never needs NCCL.
#include <nccl.h>

static thread_local char g_err[512] = "";
static std::atomic<uint64_t> g_launches{0};

extern "C" void hbgpu_set_error(const char *fmt, ...) {
    va_list ap;
    va_start(ap, fmt);
    vsnprintf(g_err, sizeof(g_err), fmt, ap);
    va_end(ap);
}

extern "C" void hbgpu_count_launch(uint64_t n) { g_launches.fetch_add(n, std::memory_order_relaxed); }

int hbgpu_check_launch(const char *what) {
    cudaError_t e = cudaGetLastError();
    if (e != cudaSuccess) {
        hbgpu_set_error("%s: %s", what, cudaGetErrorString(e));
        return HBGPU_ERR_CUDA;
    }
    return HBGPU_OK;
}

extern "C" const char *hbgpu_last_error(void) { return g_err; }
extern "C" int hbgpu_abi_version(void) { return HBGPU_ABI_VERSION; }
extern "C" uint64_t hbgpu_launch_count(void) { return g_launches.load(); }

extern "C" int hbgpu_abi_layout(int64_t *out, int32_t n) {
    const int64_t v[] = {(int64_t)sizeof(hbgpu_block),       (int64_t)sizeof(hbgpu_face_target),
                         (int64_t)sizeof(hbgpu_halo_dir),    (int64_t)sizeof(hbgpu_force_seg),
                         (int64_t)sizeof(hbgpu_peer_msg),    (int64_t)sizeof(hbgpu_stage_args),
                         (int64_t)sizeof(hbgpu_engine_desc), (int64_t)offsetof(hbgpu_engine_desc, coef),
                         (int64_t)offsetof(hbgpu_stage_args, coef), (int64_t)sizeof(hbgpu_out_record)};
    int k = 0;
    for (; k < n && k < (int)(sizeof(v) / sizeof(v[0])); ++k) out[k] = v[k];
    return k;
}

// ---- NCCL via dlopen --------------------------------------------------------

namespace {

struct NcclApi {
    bool loaded = false;
    ncclResult_t (*GetUniqueId)(ncclUniqueId *) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t *, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    ncclResult_t (*Send)(const void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void *, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void *, void *, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllReduce)(const void *, void *, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*CommGetAsyncError)(ncclComm_t, ncclResult_t *) = nullptr;
    ncclResult_t (*CommAbort)(ncclComm_t) = nullptr;
    const char *(*GetErrorString)(ncclResult_t) = nullptr;
};

NcclApi g_nccl;

bool load_nccl() {
    if (g_nccl.loaded) return true;
    void *h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) {
        hbgpu_set_error("cannot dlopen libnccl.so.2: %s", dlerror());
        return false;
    }
#define HB_SYM(field, name)                                              \
    g_nccl.field = reinterpret_cast<decltype(g_nccl.field)>(dlsym(h, name)); \
    if (!g_nccl.field) {                                                 \
        hbgpu_set_error("libnccl lacks %s", name);                       \
        return false;                                                    \
    }
    HB_SYM(GetUniqueId, "ncclGetUniqueId");
    HB_SYM(CommInitRank, "ncclCommInitRank");
    HB_SYM(CommDestroy, "ncclCommDestroy");
    HB_SYM(GroupStart, "ncclGroupStart");
    HB_SYM(GroupEnd, "ncclGroupEnd");
    HB_SYM(Send, "ncclSend");
    HB_SYM(Recv, "ncclRecv");
    HB_SYM(AllGather, "ncclAllGather");
    HB_SYM(AllReduce, "ncclAllReduce");
    HB_SYM(CommGetAsyncError, "ncclCommGetAsyncError");
    HB_SYM(CommAbort, "ncclCommAbort");
    HB_SYM(GetErrorString, "ncclGetErrorString");
#undef HB_SYM
    g_nccl.loaded = true;
    return true;
}

int nccl_fail(const char *what, ncclResult_t r) {
    hbgpu_set_error("%s: %s", what, g_nccl.GetErrorString ? g_nccl.GetErrorString(r) : "nccl error");
    return HBGPU_ERR_NCCL;
}

}  // namespace

extern "C" int hbgpu_comm_unique_id(unsigned char id[128]) {
    if (!load_nccl()) return HBGPU_ERR_NCCL;
    ncclUniqueId uid;
    ncclResult_t r = g_nccl.GetUniqueId(&uid);
    if (r != ncclSuccess) return nccl_fail("ncclGetUniqueId", r);
    memcpy(id, uid.internal, 128);
    return HBGPU_OK;
}

extern "C" int hbgpu_comm_init(const unsigned char id[128], int32_t nranks, int32_t rank, int32_t device,
                               void **comm) {
    if (!load_nccl()) return HBGPU_ERR_NCCL;
    if (cudaSetDevice(device) != cudaSuccess) return hbgpu_check_launch("cudaSetDevice");
    ncclUniqueId uid;
    memcpy(uid.internal, id, 128);
    ncclComm_t c;
    ncclResult_t r = g_nccl.CommInitRank(&c, nranks, uid, rank);
    if (r != ncclSuccess) return nccl_fail("ncclCommInitRank", r);
    *comm = (void *)c;
    return HBGPU_OK;
}

extern "C" int hbgpu_comm_allgather(void *comm, const double *send, double *recv, int64_t count,
                                    void *stream) {
    if (!load_nccl()) return HBGPU_ERR_NCCL;
    ncclResult_t r = g_nccl.AllGather(send, recv, (size_t)count, ncclFloat64, (ncclComm_t)comm,
                                      (cudaStream_t)stream);
    if (r != ncclSuccess) return nccl_fail("ncclAllGather", r);
    return HBGPU_OK;
}

extern "C" int hbgpu_comm_allreduce(void *comm, const void *send, void *recv, int64_t count, int32_t op,
                                    void *stream) {
    if (!load_nccl()) return HBGPU_ERR_NCCL;
    ncclDataType_t t;
    ncclRedOp_t o;
    if (op == HBGPU_REDUCE_SUM_F64) {
        t = ncclFloat64;
        o = ncclSum;
    } else if (op == HBGPU_REDUCE_MIN_U64) {
        t = ncclUint64;
        o = ncclMin;
    } else {
        hbgpu_set_error("hbgpu_comm_allreduce: unknown op %d", op);
        return HBGPU_ERR_ARG;
    }
    ncclResult_t r = g_nccl.AllReduce(send, recv, (size_t)count, t, o, (ncclComm_t)comm, (cudaStream_t)stream);
    if (r != ncclSuccess) return nccl_fail("ncclAllReduce", r);
    return HBGPU_OK;
}

extern "C" int hbgpu_comm_exchange(void *comm, const double *sendbuf, const hbgpu_peer_msg *sends, int32_t nsends,
                                   double *recvbuf, const hbgpu_peer_msg *recvs, int32_t nrecvs, void *stream) {
    if (!load_nccl()) return HBGPU_ERR_NCCL;
    if (comm == nullptr || nsends < 0 || nrecvs < 0) {
        hbgpu_set_error("hbgpu_comm_exchange: bad arguments");
        return HBGPU_ERR_ARG;
    }
    cudaStream_t s = (cudaStream_t)stream;
    ncclResult_t r = g_nccl.GroupStart();
    if (r != ncclSuccess) return nccl_fail("ncclGroupStart", r);
    for (int k = 0; k < nsends; ++k) {
        r = g_nccl.Send(sendbuf + sends[k].offset, (size_t)sends[k].count, ncclFloat64, sends[k].peer,
                        (ncclComm_t)comm, s);
        if (r != ncclSuccess) return nccl_fail("ncclSend", r);
    }
    for (int k = 0; k < nrecvs; ++k) {
        r = g_nccl.Recv(recvbuf + recvs[k].offset, (size_t)recvs[k].count, ncclFloat64, recvs[k].peer,
                        (ncclComm_t)comm, s);
        if (r != ncclSuccess) return nccl_fail("ncclRecv", r);
    }
    r = g_nccl.GroupEnd();
    if (r != ncclSuccess) return nccl_fail("ncclGroupEnd", r);
    return HBGPU_OK;
}

extern "C" int hbgpu_comm_async_error(void *comm) {
    if (comm == nullptr) return HBGPU_OK;
    if (!load_nccl()) return HBGPU_ERR_NCCL;
    ncclResult_t err = ncclSuccess;
    ncclResult_t r = g_nccl.CommGetAsyncError((ncclComm_t)comm, &err);
    if (r != ncclSuccess) return nccl_fail("ncclCommGetAsyncError", r);
    if (err != ncclSuccess && err != ncclInProgress) return nccl_fail("NCCL asynchronous error", err);
    return HBGPU_OK;
}

extern "C" int hbgpu_comm_abort(void *comm) {
    if (comm == nullptr) return HBGPU_OK;
    if (!load_nccl()) return HBGPU_ERR_NCCL;
    ncclResult_t r = g_nccl.CommAbort((ncclComm_t)comm);
    if (r != ncclSuccess) return nccl_fail("ncclCommAbort", r);
    return HBGPU_OK;
}

extern "C" int hbgpu_comm_destroy(void *comm) {
    if (comm == nullptr) return HBGPU_OK;
    if (!load_nccl()) return HBGPU_ERR_NCCL;
    ncclResult_t r = g_nccl.CommDestroy((ncclComm_t)comm);
    if (r != ncclSuccess) return nccl_fail("ncclCommDestroy", r);
    return HBGPU_OK;
}

// ---- engine -------------------------------------------------------------------

struct hbgpu_engine {
    hbgpu_engine_desc d;
    cudaStream_t work = nullptr;
    cudaEvent_t ev_in = nullptr, ev_out = nullptr;
    std::vector<hbgpu_peer_msg> sends, recvs;
    cudaGraph_t graph = nullptr;
    cudaGraphExec_t exec = nullptr;
    bool graph_failed = false;   // capture or instantiation failed once: eager iterations from then on
    int32_t done = 0;   // iterations issued (rows of sumsq / force_hist used)
    // multi-GPU overlap: boundary tiles -> remote pack -> NCCL on `comm_s`
    // while the interior tiles run on the work stream (run_split)
    bool split = false;
    cudaStream_t comm_s = nullptr;
    cudaEvent_t ev_pack = nullptr, ev_comm = nullptr;
    // the stage-0 norm fold runs on aux_s, off the critical path: forked
    // after the first pass, joined before the forces (which advance the
    // iteration counter the fold reads); captured into the graph as a branch
    cudaStream_t aux_s = nullptr;
    cudaEvent_t ev_nf_fork = nullptr, ev_nf_join = nullptr;
    // small schedule: per-warp-task stage-0 partials of the cooperative kernel
    double *small_part = nullptr;
    int small_tasks = 0;
};

namespace hbgpu {
int small_prepare(const hbgpu_engine_desc &d, int *tasks, double **part_buf);
int small_iterations(const hbgpu_engine_desc &d, int32_t it0, int32_t iters, cudaStream_t s, double *part_buf,
                     int tasks);
}

namespace {

// slot rotation per stage: (in, out); q0 is always slot 0 (A).
//   stage 0: A -> B, stage 1: B -> C, stage 2: C -> B, stage 3: B -> A (in place on q0)
constexpr int kIn[4] = {0, 1, 2, 1};
constexpr int kOut[4] = {1, 2, 1, 0};

// one grouped NCCL send/recv of every peer segment (exchange.py:307-316:
// one aggregated message per direction, here per peer) on stream s
int nccl_group(hbgpu_engine *e, cudaStream_t s) {
    const hbgpu_engine_desc &d = e->d;
    if (!load_nccl()) return HBGPU_ERR_NCCL;
    ncclComm_t comm = (ncclComm_t)d.comm;
    ncclResult_t r = g_nccl.GroupStart();
    if (r != ncclSuccess) return nccl_fail("ncclGroupStart", r);
    for (const auto &m : e->sends) {
        r = g_nccl.Send(d.sendbuf + m.offset, (size_t)m.count, ncclFloat64, m.peer, comm, s);
        if (r != ncclSuccess) return nccl_fail("ncclSend", r);
    }
    for (const auto &m : e->recvs) {
        r = g_nccl.Recv(d.recvbuf + m.offset, (size_t)m.count, ncclFloat64, m.peer, comm, s);
        if (r != ncclSuccess) return nccl_fail("ncclRecv", r);
    }
    r = g_nccl.GroupEnd();
    if (r != ncclSuccess) return nccl_fail("ncclGroupEnd", r);
    return HBGPU_OK;
}

int exchange_remote(hbgpu_engine *e, double *slot, cudaStream_t s) {
    const hbgpu_engine_desc &d = e->d;
    if (d.comm == nullptr || (e->sends.empty() && e->recvs.empty())) return HBGPU_OK;
    if (!load_nccl()) return HBGPU_ERR_NCCL;
    ncclComm_t comm = (ncclComm_t)d.comm;
    ncclResult_t r = g_nccl.GroupStart();
    if (r != ncclSuccess) return nccl_fail("ncclGroupStart", r);
    for (const auto &m : e->sends) {
        r = g_nccl.Send(d.sendbuf + m.offset, (size_t)m.count, ncclFloat64, m.peer, comm, s);
        if (r != ncclSuccess) return nccl_fail("ncclSend", r);
    }
    for (const auto &m : e->recvs) {
        r = g_nccl.Recv(d.recvbuf + m.offset, (size_t)m.count, ncclFloat64, m.peer, comm, s);
        if (r != ncclSuccess) return nccl_fail("ncclRecv", r);
    }
    r = g_nccl.GroupEnd();
    if (r != ncclSuccess) return nccl_fail("ncclGroupEnd", r);
    return hbgpu_halo(slot, d.sendbuf, d.recvbuf, d.unpack_dirs, d.nunpack, d.unpack_max_len, d.planes, s);
}

// fused (paired) schedule, per phase: (stencil slot, output slot)
//   0: band(0)     A -> C (perimeter cells + halos)
//   1: pair(0, 1)  A (+ band C) -> B
//   2: band(2)     B, base A -> C
//   3: pair(2, 3)  B, base A (+ band C) -> A, then a full halo pass on A
constexpr int kInF[4] = {0, 0, 1, 1};
constexpr int kOutF[4] = {2, 1, 2, 0};

inline int out_slot(const hbgpu_engine_desc &d, int phase) { return d.fused ? kOutF[phase] : kOut[phase]; }

void fill_args(const hbgpu_engine_desc &d, hbgpu_stage_args &a) {
    memset(&a, 0, sizeof(a));
    a.q0 = d.slot[0];
    a.band = d.slot[2];
    a.sendbuf = d.sendbuf;
    a.blocks = d.blocks;
    a.tile_block = d.tile_block;
    a.sxy = d.sxy;
    a.faces = d.faces;
    a.status = d.status;
    a.iter = d.iter;
    a.dmat = d.dmat;
    a.tmaps = d.tmaps;
    a.nblocks = d.nblocks;
    a.total_tiles = d.total_tiles;
    a.planes = d.planes;
    a.tile_rows = d.tile_rows;
    a.interleaved = d.interleaved;
    a.tile_pdes = d.tile_pdes;
    a.band_segs = d.band_segs;
    a.nband_segs = d.nband_segs;
    a.band_max_len = d.band_max_len;
    a.edge_q0 = d.edge_q0;
    memcpy(a.D, d.D, sizeof(a.D));
    memcpy(a.ap, d.ap, sizeof(a.ap));
}

// arguments of phase `ph` of the paired schedule (hb_pair.cu)
void fused_args(const hbgpu_engine_desc &d, int ph, hbgpu_stage_args &a) {
    fill_args(d, a);
    const int st = ph < 2 ? 0 : 2;   // the first stage of the pair
    a.in = d.slot[kInF[ph]];
    a.in_slot = kInF[ph];
    a.out = d.slot[kOutF[ph]];
    a.out_slot = kOutF[ph];
    a.stage = st;
    a.coef = d.coef[st];
    if (ph == 1 || ph == 3) {
        a.pair = ph == 1 ? 1 : 2;
        a.coef2 = d.coef[st + 1];
        a.norm_part = ph == 1 ? d.norm_part : nullptr;
    }
}

// arguments of single RK stage `st` (hb_stage.cu)
void single_args(const hbgpu_engine_desc &d, int st, hbgpu_stage_args &a) {
    fill_args(d, a);
    a.band = nullptr;
    a.band_segs = nullptr;
    a.nband_segs = 0;
    a.band_max_len = 0;
    a.edge_q0 = nullptr;
    a.in = d.slot[kIn[st]];
    a.out = d.slot[kOut[st]];
    a.stage = st;
    a.in_slot = kIn[st];
    a.out_slot = kOut[st];
    a.coef = d.coef[st];
    a.norm_part = st == 0 ? d.norm_part : nullptr;
}

// The halo moves that follow a stage kernel, split in the remote packs
// (the first `remote` of `dirs`, dst_kind 1) and the local copies:
//   pass A, and single stage 0 unless it forwards them itself
//   (hbgpu_stage_first_forwards): west / east face columns (post_dirs);
//   pass B: the full halo pass (prime_dirs), pass B forwarding nothing
//   itself because it writes q4 over q0, which other tiles still read.
struct PostMoves {
    const hbgpu_halo_dir *dirs = nullptr;
    int32_t n = 0, remote = 0, max_len = 0;
};

PostMoves post_moves(const hbgpu_engine_desc &d, int st) {
    PostMoves m;
    if (d.fused ? st == 1 : (st == 0 && !hbgpu_stage_first_forwards(d.planes))) {
        m.dirs = d.post_dirs;
        m.n = d.npost;
        m.remote = d.post_remote;
        m.max_len = d.post_max_len;
    } else if (d.fused && st == 3) {
        m.dirs = d.prime_dirs;
        m.n = d.nprime;
        m.remote = d.prime_remote;
        m.max_len = d.prime_max_len;
    }
    return m;
}

int halo_moves(const hbgpu_engine_desc &d, double *slot, const hbgpu_halo_dir *dirs, int32_t n, int32_t max_len,
               cudaStream_t s) {
    if (n <= 0) return HBGPU_OK;
    return hbgpu_halo(slot, d.sendbuf, d.recvbuf, dirs, n, max_len, d.planes, s);
}

// stage / phase `st` (+ the norm fold after the first stage, + its halo moves).
// fork_norm: the norm fold goes to aux_s (joined by join_norm) instead of
// between the pass and its halo moves.
int run_stage(hbgpu_engine *e, int st, cudaStream_t s, bool fork_norm = false) {
    const hbgpu_engine_desc &d = e->d;
    hbgpu_stage_args a;
    if (d.fused) fused_args(d, st, a);
    else single_args(d, st, a);
    if (d.fused && (st == 0 || st == 2)) return hbgpu_band(&a, s);
    int rc = hbgpu_stage(&a, s);
    if (!rc && a.norm_part != nullptr) {
        if (fork_norm) {
            if (cudaEventRecord(e->ev_nf_fork, s) != cudaSuccess ||
                cudaStreamWaitEvent(e->aux_s, e->ev_nf_fork, 0) != cudaSuccess)
                return hbgpu_check_launch("norm fold fork");
            rc = hbgpu_norm_fold(d.blocks, d.nblocks, d.norm_part, d.sumsq, d.iter, d.max_iters, e->aux_s);
            if (!rc && cudaEventRecord(e->ev_nf_join, e->aux_s) != cudaSuccess)
                rc = hbgpu_check_launch("norm fold record");
        } else {
            rc = hbgpu_norm_fold(d.blocks, d.nblocks, d.norm_part, d.sumsq, d.iter, d.max_iters, s);
        }
    }
    const PostMoves m = post_moves(d, st);
    if (!rc) rc = halo_moves(d, a.out, m.dirs, m.n, m.max_len, s);
    return rc;
}

// The same stage with its remote exchange overlapped (multi-GPU):
//   work:   boundary tiles -> remote packs -> [ev_pack] -> interior tiles ->
//           norm fold -> local halo copies -> wait [ev_comm] -> unpack
//   comm_s: wait [ev_pack] -> ncclGroupStart / Send / Recv / End -> [ev_comm]
// Boundary tiles hold every cell this rank sends (devlayout tile_order), so
// the send buffer is complete at ev_pack; interior tiles neither write a
// sent cell nor read a received halo, so they may run under the transfer;
// the unpack writes the received halos once both are done.  Band phases
// (all perimeter work) exchange after the kernel as before.
int split_part(hbgpu_engine *e, int st, int part, cudaStream_t s) {
    const hbgpu_engine_desc &d = e->d;
    hbgpu_stage_args a;
    if (d.fused) fused_args(d, st, a);
    else single_args(d, st, a);
    const PostMoves m = post_moves(d, st);
    a.tile_order = d.tile_order;
    if (part == 0) {   // boundary tiles, then the remote packs
        a.tile_lo = 0;
        a.tile_hi = d.nbound_tiles;
        int rc = hbgpu_stage(&a, s);
        if (!rc) rc = halo_moves(d, a.out, m.dirs, m.remote, m.max_len, s);
        return rc;
    }
    // interior tiles, the norm fold (first stage), the local halo copies
    a.tile_lo = d.nbound_tiles;
    a.tile_hi = d.total_tiles;
    int rc = hbgpu_stage(&a, s);
    if (!rc && a.norm_part != nullptr)
        rc = hbgpu_norm_fold(d.blocks, d.nblocks, d.norm_part, d.sumsq, d.iter, d.max_iters, s);
    if (!rc) rc = halo_moves(d, a.out, m.dirs + m.remote, m.n - m.remote, m.max_len, s);
    return rc;
}

int run_split(hbgpu_engine *e, int st, cudaStream_t s) {
    const hbgpu_engine_desc &d = e->d;
    int rc = split_part(e, st, 0, s);
    if (!rc && (cudaEventRecord(e->ev_pack, s) != cudaSuccess ||
                cudaStreamWaitEvent(e->comm_s, e->ev_pack, 0) != cudaSuccess))
        rc = hbgpu_check_launch("run_split fork");
    if (!rc) rc = nccl_group(e, e->comm_s);
    if (!rc && cudaEventRecord(e->ev_comm, e->comm_s) != cudaSuccess) rc = hbgpu_check_launch("run_split record");
    if (!rc) rc = split_part(e, st, 1, s);
    if (!rc && cudaStreamWaitEvent(s, e->ev_comm, 0) != cudaSuccess) rc = hbgpu_check_launch("run_split join");
    if (!rc) rc = halo_moves(d, d.slot[out_slot(d, st)], d.unpack_dirs, d.nunpack, d.unpack_max_len, s);
    return rc;
}

// a pass (stage kernel) phase, as opposed to a band phase
inline bool pass_phase(const hbgpu_engine_desc &d, int st) { return !d.fused || st == 1 || st == 3; }

int one_iteration(hbgpu_engine *e, cudaStream_t s) {
    const hbgpu_engine_desc &d = e->d;
    for (int st = 0; st < 4; ++st) {
        int rc;
        if (e->split && pass_phase(d, st)) {
            rc = run_split(e, st, s);
        } else {
            rc = run_stage(e, st, s, true);
            if (!rc) rc = exchange_remote(e, d.slot[out_slot(d, st)], s);
        }
        if (rc) return rc;
    }
    // join the forked norm fold (no-op when the fold ran in line)
    if (!e->split && cudaStreamWaitEvent(s, e->ev_nf_join, 0) != cudaSuccess)
        return hbgpu_check_launch("norm fold join");
    return hbgpu_forces(d.slot[0], d.segs, d.nsegs, d.planes, d.nbody, d.force_hist, d.iter, d.max_iters, s);
}

// the sumsq / force_hist rows the next `n` iterations would use exist
int check_capacity(const hbgpu_engine *e, int64_t n, const char *who) {
    if (n < 0 || (int64_t)e->done + n > (int64_t)e->d.max_iters) {
        hbgpu_set_error("%s: %lld more iteration(s) after %d would exceed max_iters = %d (the capacity of "
                        "sumsq and force_hist); rewind or create the engine with a larger max_iters",
                        who, (long long)n, e->done, e->d.max_iters);
        return HBGPU_ERR_ARG;
    }
    return HBGPU_OK;
}

}  // namespace

extern "C" int hbgpu_engine_create(const hbgpu_engine_desc *desc, hbgpu_engine **out) {
    if (desc == nullptr || out == nullptr || desc->planes < 1 || desc->nblocks < 1) {
        hbgpu_set_error("hbgpu_engine_create: bad descriptor");
        return HBGPU_ERR_ARG;
    }
    if (desc->fused && desc->edge_q0 == nullptr) {
        hbgpu_set_error("hbgpu_engine_create: fused schedule needs edge_q0");
        return HBGPU_ERR_ARG;
    }
    if (desc->small && (desc->fused || desc->nsends > 0 || desc->nrecvs > 0 || desc->small_max_cells <= 0 ||
                        desc->planes > 9 || desc->planes % 2 == 0)) {
        hbgpu_set_error("hbgpu_engine_create: the small schedule needs one rank without remote cuts, single "
                        "stages, P <= 9 and small_max_cells");
        return HBGPU_ERR_ARG;
    }
    int prc = hbgpu_stage_prepare(desc->planes);
    if (prc) return prc;
    auto *e = new hbgpu_engine();
    e->d = *desc;
    if (desc->nsends > 0) e->sends.assign(desc->sends, desc->sends + desc->nsends);
    if (desc->nrecvs > 0) e->recvs.assign(desc->recvs, desc->recvs + desc->nrecvs);
    e->d.sends = nullptr;
    e->d.recvs = nullptr;
    if (cudaStreamCreateWithFlags(&e->work, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_in, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_out, cudaEventDisableTiming) != cudaSuccess ||
        cudaStreamCreateWithFlags(&e->aux_s, cudaStreamNonBlocking) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_nf_fork, cudaEventDisableTiming) != cudaSuccess ||
        cudaEventCreateWithFlags(&e->ev_nf_join, cudaEventDisableTiming) != cudaSuccess) {
        int rc = hbgpu_check_launch("hbgpu_engine_create");
        hbgpu_engine_destroy(e);
        return rc ? rc : HBGPU_ERR_CUDA;
    }
    // overlap the remote exchange of every pass with its interior tiles when
    // this rank sends and has a boundary/interior tile split to use
    e->split = desc->comm != nullptr && !e->sends.empty() && desc->tile_order != nullptr &&
               desc->nbound_tiles > 0 && desc->nbound_tiles < desc->total_tiles;
    if (e->split && (cudaStreamCreateWithFlags(&e->comm_s, cudaStreamNonBlocking) != cudaSuccess ||
                     cudaEventCreateWithFlags(&e->ev_pack, cudaEventDisableTiming) != cudaSuccess ||
                     cudaEventCreateWithFlags(&e->ev_comm, cudaEventDisableTiming) != cudaSuccess)) {
        int rc = hbgpu_check_launch("hbgpu_engine_create (comm stream)");
        hbgpu_engine_destroy(e);
        return rc ? rc : HBGPU_ERR_CUDA;
    }
    if (desc->small) {
        int rc = hbgpu::small_prepare(e->d, &e->small_tasks, &e->small_part);
        if (rc) {
            hbgpu_engine_destroy(e);
            return rc;
        }
    }
    *out = e;
    return HBGPU_OK;
}

namespace {
// caller stream -> engine stream ordering on entry, and back on exit
int enter(hbgpu_engine *e, cudaStream_t caller) {
    if (cudaEventRecord(e->ev_in, caller) != cudaSuccess ||
        cudaStreamWaitEvent(e->work, e->ev_in, 0) != cudaSuccess)
        return hbgpu_check_launch("hbgpu_engine enter");
    return HBGPU_OK;
}
int leave(hbgpu_engine *e, cudaStream_t caller, int rc) {
    if (cudaEventRecord(e->ev_out, e->work) != cudaSuccess ||
        cudaStreamWaitEvent(caller, e->ev_out, 0) != cudaSuccess) {
        int lrc = hbgpu_check_launch("hbgpu_engine leave");
        return rc ? rc : lrc;
    }
    return rc;
}
}  // namespace

extern "C" int hbgpu_engine_prime(hbgpu_engine *e, void *stream) {
    cudaStream_t caller = (cudaStream_t)stream;
    int rc = enter(e, caller);
    if (rc) return rc;
    const hbgpu_engine_desc &d = e->d;
    // the paired kernel's exact rewrites need |q| < 2^1022 in its inputs
    if (d.fused) rc = hbgpu_hazard_scan(d.slot[0], d.blocks, d.nblocks, d.planes, d.status, e->work);
    if (!rc)
        rc = hbgpu_halo(d.slot[0], d.sendbuf, d.recvbuf, d.prime_dirs, d.nprime, d.prime_max_len, d.planes,
                        e->work);
    if (!rc) rc = exchange_remote(e, d.slot[0], e->work);
    return leave(e, caller, rc);
}

// ---- stepwise schedule: the same iteration split at its exchange points, for
// callers that move the remote halo payloads themselves (one process driving
// several ranks' engines, e.g. the loopback transport of solver.run_case).
// phase: -1 = priming exchange (halo kernel: local copies + pack of slot A),
//        0..3 = fused stage kernel of that RK stage (+ norm fold after 0),
//        4 = forces + iteration counter.
// unpack(e, phase) scatters the receive buffer into the slot phase wrote.

extern "C" int hbgpu_engine_step(hbgpu_engine *e, int32_t phase, void *stream) {
    cudaStream_t caller = (cudaStream_t)stream;
    int rc = enter(e, caller);
    if (rc) return rc;
    const hbgpu_engine_desc &d = e->d;
    if (phase == -1) {
        if (d.fused) rc = hbgpu_hazard_scan(d.slot[0], d.blocks, d.nblocks, d.planes, d.status, e->work);
        if (!rc)
            rc = hbgpu_halo(d.slot[0], d.sendbuf, d.recvbuf, d.prime_dirs, d.nprime, d.prime_max_len, d.planes,
                            e->work);
    }
    else if (phase >= 0 && phase < 4)
        rc = run_stage(e, phase, e->work);
    else if (phase == 4) {
        rc = check_capacity(e, 1, "hbgpu_engine_step");
        if (!rc) rc = hbgpu_forces(d.slot[0], d.segs, d.nsegs, d.planes, d.nbody, d.force_hist, d.iter,
                                   d.max_iters, e->work);
        if (!rc) ++e->done;
    }
    else {
        hbgpu_set_error("hbgpu_engine_step: bad phase %d", phase);
        rc = HBGPU_ERR_ARG;
    }
    return leave(e, caller, rc);
}

extern "C" int hbgpu_engine_step_split(hbgpu_engine *e, int32_t phase, int32_t part, void *stream) {
    const hbgpu_engine_desc &d = e->d;
    if (phase < 0 || phase > 3 || part < 0 || part > 1 || !pass_phase(d, phase) || d.tile_order == nullptr) {
        hbgpu_set_error("hbgpu_engine_step_split: phase %d part %d is not a split pass phase (or no tile_order)",
                        phase, part);
        return HBGPU_ERR_ARG;
    }
    cudaStream_t caller = (cudaStream_t)stream;
    int rc = enter(e, caller);
    if (rc) return rc;
    rc = split_part(e, phase, part, e->work);
    return leave(e, caller, rc);
}

extern "C" int hbgpu_engine_unpack(hbgpu_engine *e, int32_t phase, void *stream) {
    cudaStream_t caller = (cudaStream_t)stream;
    if (phase < -1 || phase > 3) {
        hbgpu_set_error("hbgpu_engine_unpack: bad phase %d", phase);
        return HBGPU_ERR_ARG;
    }
    int rc = enter(e, caller);
    if (rc) return rc;
    const hbgpu_engine_desc &d = e->d;
    double *slot = phase < 0 ? d.slot[0] : d.slot[out_slot(d, phase)];
    rc = hbgpu_halo(slot, d.sendbuf, d.recvbuf, d.unpack_dirs, d.nunpack, d.unpack_max_len, d.planes, e->work);
    return leave(e, caller, rc);
}

extern "C" int hbgpu_engine_launches_per_iteration(const hbgpu_engine *e) {
    const hbgpu_engine_desc &d = e->d;
    if (d.small) return 1;   // one cooperative launch per hbgpu_engine_iterate call (<= 1 per iteration)
    const bool remote = d.comm != nullptr && !e->recvs.empty() && d.nunpack > 0;
    int n = 1;   // forces
    for (int st = 0; st < 4; ++st) {
        const PostMoves m = post_moves(d, st);
        const bool fold = d.fused ? st == 1 : st == 0;
        if (e->split && pass_phase(d, st)) {
            n += 2 + (fold ? 1 : 0) + (m.remote > 0 ? 1 : 0) + (m.n - m.remote > 0 ? 1 : 0) + (remote ? 1 : 0);
        } else {
            n += 1 + (pass_phase(d, st) && fold ? 1 : 0) + (m.n > 0 ? 1 : 0) + (remote ? 1 : 0);
        }
    }
    return n;
}

static int iterate_on(hbgpu_engine *e, int32_t iterations, int32_t use_graph, cudaStream_t s);

extern "C" int hbgpu_engine_iterate(hbgpu_engine *e, int32_t iterations, int32_t use_graph, void *stream) {
    if (e == nullptr) {
        hbgpu_set_error("hbgpu_engine_iterate: null engine");
        return HBGPU_ERR_ARG;
    }
    int rc = check_capacity(e, iterations, "hbgpu_engine_iterate");
    if (rc) return rc;
    cudaStream_t caller = (cudaStream_t)stream;
    rc = enter(e, caller);
    if (rc) return rc;
    if (e->d.small)
        rc = hbgpu::small_iterations(e->d, e->done, iterations, e->work, e->small_part, e->small_tasks);
    else
        rc = iterate_on(e, iterations, use_graph, e->work);
    if (!rc) e->done += iterations;
    return leave(e, caller, rc);
}

extern "C" int hbgpu_engine_iterations_done(const hbgpu_engine *e) { return e ? e->done : 0; }

extern "C" int hbgpu_engine_rewind(hbgpu_engine *e, void *stream) {
    if (e == nullptr) {
        hbgpu_set_error("hbgpu_engine_rewind: null engine");
        return HBGPU_ERR_ARG;
    }
    cudaStream_t caller = (cudaStream_t)stream;
    int rc = enter(e, caller);
    if (rc) return rc;
    if (cudaMemsetAsync(e->d.iter, 0, sizeof(int32_t), e->work) != cudaSuccess ||
        cudaMemsetAsync(e->d.status, 0xff, sizeof(unsigned long long) * (size_t)e->d.nblocks, e->work) !=
            cudaSuccess)
        rc = hbgpu_check_launch("hbgpu_engine_rewind");
    if (!rc) e->done = 0;
    return leave(e, caller, rc);
}

static int iterate_on(hbgpu_engine *e, int32_t iterations, int32_t use_graph, cudaStream_t s) {
    if (!use_graph || e->graph_failed) {
        for (int it = 0; it < iterations; ++it) {
            int rc = one_iteration(e, s);
            if (rc) return rc;
        }
        return HBGPU_OK;
    }
    if (e->exec == nullptr) {
        cudaError_t ce = cudaStreamBeginCapture(s, cudaStreamCaptureModeThreadLocal);
        if (ce != cudaSuccess) {
            hbgpu_set_error("cudaStreamBeginCapture: %s", cudaGetErrorString(ce));
            return HBGPU_ERR_CUDA;
        }
        uint64_t before = g_launches.load();
        int rc = one_iteration(e, s);
        cudaGraph_t g = nullptr;
        ce = cudaStreamEndCapture(s, &g);
        // captured launches are counted when the graph replays
        g_launches.store(before);
        if (!rc && ce == cudaSuccess) ce = cudaGraphInstantiate(&e->exec, g, 0);
        if (rc || ce != cudaSuccess) {
            // Nothing of the iteration has run (it was only being recorded).
            // An operation that cannot be captured -- e.g. a collective of a
            // communicator library that refuses stream capture -- must not
            // end the run: this engine issues its iterations eagerly from now
            // on; a real error shows again there and is returned.
            if (g) cudaGraphDestroy(g);
            e->exec = nullptr;
            cudaGetLastError();
            e->graph_failed = true;
            return iterate_on(e, iterations, 0, s);
        }
        e->graph = g;
    }
    const int per_it = hbgpu_engine_launches_per_iteration(e);
    for (int it = 0; it < iterations; ++it) {
        cudaError_t ce = cudaGraphLaunch(e->exec, s);
        if (ce != cudaSuccess) {
            hbgpu_set_error("cudaGraphLaunch: %s", cudaGetErrorString(ce));
            return HBGPU_ERR_CUDA;
        }
        hbgpu_count_launch(per_it);
    }
    return HBGPU_OK;
}

extern "C" int hbgpu_engine_destroy(hbgpu_engine *e) {
    if (e == nullptr) return HBGPU_OK;
    if (e->exec) cudaGraphExecDestroy(e->exec);
    if (e->graph) cudaGraphDestroy(e->graph);
    if (e->work) {
        cudaStreamSynchronize(e->work);
        cudaStreamDestroy(e->work);
    }
    if (e->ev_in) cudaEventDestroy(e->ev_in);
    if (e->ev_out) cudaEventDestroy(e->ev_out);
    if (e->comm_s) {
        cudaStreamSynchronize(e->comm_s);
        cudaStreamDestroy(e->comm_s);
    }
    if (e->ev_pack) cudaEventDestroy(e->ev_pack);
    if (e->ev_comm) cudaEventDestroy(e->ev_comm);
    if (e->aux_s) {
        cudaStreamSynchronize(e->aux_s);
        cudaStreamDestroy(e->aux_s);
    }
    if (e->ev_nf_fork) cudaEventDestroy(e->ev_nf_fork);
    if (e->ev_nf_join) cudaEventDestroy(e->ev_nf_join);
    if (e->small_part) cudaFree(e->small_part);
    delete e;
    return HBGPU_OK;
}
