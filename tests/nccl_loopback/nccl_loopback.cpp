// nccl_loopback.cpp -- TEST INFRASTRUCTURE: an in-process stand-in for the
// handful of NCCL entry points libmfx uses (GetUniqueId, CommInitRank,
// CommDestroy, CommSplit, GroupStart/End, Send, Recv, Broadcast, AllGather,
// GetErrorString), so that libmfx's NCCL transport -- the code path a real
// multi-GPU run takes (simple.cu: exchange_state / ctx_halo_exchange /
// ctx_allgather_dd on communicators and a split sub-communicator) -- can run
// with thread-ranks on the single GPU of a gpurun box, where real NCCL refuses
// two ranks on one device.  libmfx loads it through MFX_NCCL_PATH.
//
// Semantics follow NCCL's: operations inside a group are issued together;
// point-to-point messages between a pair match in issue order; collectives
// match in issue order on a communicator.  Data moves with cudaMemcpyAsync on
// the caller's stream, ordered by events: a receiver's stream waits for the
// sender's "ready" event, the copy is enqueued, and the sender's stream waits
// for the receiver's "done" event (the buffer is reusable once delivered).
// The host blocks inside GroupEnd until the peers have posted (so this shim
// must not be used under CUDA-graph capture: MFX_DIST_GRAPH=0).
#include <cuda_runtime.h>
#include <nccl.h>

#include <algorithm>
#include <condition_variable>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

namespace {

struct Msg {
    const void *ptr = nullptr;
    size_t bytes = 0;
    cudaEvent_t ready = nullptr;
    cudaEvent_t done = nullptr;
    bool taken = false, delivered = false;
};

struct Coll {                       // one collective instance on a communicator
    int posted = 0, finished = 0;
    std::vector<const void *> src;  // per rank (AllGather chunk / Broadcast root buffer)
    std::vector<cudaEvent_t> ready, done;
    std::vector<int> color, key;    // CommSplit
    std::map<int, struct World *> split_worlds;
};

struct World {
    int n;
    std::mutex mu;
    std::condition_variable cv;
    std::map<std::pair<int, int>, std::deque<std::shared_ptr<Msg>>> box;   // (src, dst) FIFO
    std::map<long, Coll> coll;                                             // by sequence number
    std::vector<bool> joined;
    explicit World(int n_) : n(n_), joined(n_, false) {}
};

std::mutex g_mu;
std::map<std::string, World *> g_worlds;

}  // namespace

struct ncclComm {
    World *w;
    int rank, n;
    long seq = 0;   // collective sequence on this communicator (same on every rank)
};

namespace {

enum OpKind { SEND, RECV, BCAST, ALLGATHER };
struct Op {
    OpKind kind;
    const void *sbuf;
    void *rbuf;
    size_t bytes;
    int peer;
    ncclComm_t comm;
    cudaStream_t stream;
    long seq;
    std::shared_ptr<Msg> msg;
};
thread_local int t_depth = 0;
thread_local std::vector<Op> t_ops;

size_t dsize(ncclDataType_t t)
{
    switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
    }
}

cudaEvent_t record(cudaStream_t s)
{
    cudaEvent_t e;
    cudaEventCreateWithFlags(&e, cudaEventDisableTiming);
    cudaEventRecord(e, s);
    return e;
}

ncclResult_t run_group(std::vector<Op> &ops)
{
    // phase 1: post everything this rank provides
    for (Op &o : ops) {
        World *w = o.comm->w;
        std::unique_lock<std::mutex> lk(w->mu);
        if (o.kind == SEND) {
            o.msg = std::make_shared<Msg>();
            o.msg->ptr = o.sbuf;
            o.msg->bytes = o.bytes;
            o.msg->ready = record(o.stream);
            w->box[{o.comm->rank, o.peer}].push_back(o.msg);
        } else if (o.kind == BCAST || o.kind == ALLGATHER) {
            Coll &c = w->coll[o.seq];
            if (c.src.empty()) { c.src.assign(w->n, nullptr); c.ready.assign(w->n, nullptr); c.done.assign(w->n, nullptr); }
            const bool provides = o.kind == ALLGATHER || o.peer == o.comm->rank;
            if (provides) {
                c.src[o.comm->rank] = o.sbuf;
                c.ready[o.comm->rank] = record(o.stream);
            }
            c.posted++;
        }
        w->cv.notify_all();
    }
    // phase 2: take what this rank receives
    for (Op &o : ops) {
        World *w = o.comm->w;
        std::unique_lock<std::mutex> lk(w->mu);
        if (o.kind == RECV) {
            auto &q = w->box[{o.peer, o.comm->rank}];
            std::shared_ptr<Msg> m;
            w->cv.wait(lk, [&] {
                for (auto &x : q)
                    if (!x->taken) { m = x; return true; }
                return false;
            });
            m->taken = true;
            lk.unlock();
            if (m->bytes != o.bytes) return ncclInvalidArgument;
            cudaStreamWaitEvent(o.stream, m->ready, 0);
            cudaMemcpyAsync(o.rbuf, m->ptr, o.bytes, cudaMemcpyDefault, o.stream);
            cudaEvent_t d = record(o.stream);
            lk.lock();
            m->done = d;
            m->delivered = true;
            w->cv.notify_all();
        } else if (o.kind == BCAST || o.kind == ALLGATHER) {
            Coll &c = w->coll[o.seq];
            w->cv.wait(lk, [&] { return c.posted == w->n; });
            lk.unlock();
            if (o.kind == BCAST) {
                const int root = o.peer;
                if (root != o.comm->rank) {
                    cudaStreamWaitEvent(o.stream, c.ready[root], 0);
                    cudaMemcpyAsync(o.rbuf, c.src[root], o.bytes, cudaMemcpyDefault, o.stream);
                } else if (o.rbuf != o.sbuf) {
                    cudaMemcpyAsync(o.rbuf, o.sbuf, o.bytes, cudaMemcpyDefault, o.stream);
                }
            } else {
                for (int r = 0; r < w->n; r++) {
                    if (r != o.comm->rank) cudaStreamWaitEvent(o.stream, c.ready[r], 0);
                    cudaMemcpyAsync((char *)o.rbuf + (size_t)r * o.bytes, c.src[r], o.bytes, cudaMemcpyDefault,
                                    o.stream);
                }
            }
            cudaEvent_t d = record(o.stream);
            lk.lock();
            c.done[o.comm->rank] = d;
            c.finished++;
            w->cv.notify_all();
        }
    }
    // phase 3: this rank's stream waits until what it provided has been taken
    for (Op &o : ops) {
        World *w = o.comm->w;
        std::unique_lock<std::mutex> lk(w->mu);
        if (o.kind == SEND) {
            w->cv.wait(lk, [&] { return o.msg->delivered; });
            cudaStreamWaitEvent(o.stream, o.msg->done, 0);
            auto &q = w->box[{o.comm->rank, o.peer}];
            while (!q.empty() && q.front()->delivered) q.pop_front();
        } else if (o.kind == BCAST || o.kind == ALLGATHER) {
            Coll &c = w->coll[o.seq];
            w->cv.wait(lk, [&] { return c.finished == w->n; });
            const bool provides = o.kind == ALLGATHER || o.peer == o.comm->rank;
            if (provides)
                for (int r = 0; r < w->n; r++)
                    if (r != o.comm->rank) cudaStreamWaitEvent(o.stream, c.done[r], 0);
        }
    }
    return ncclSuccess;
}

ncclResult_t submit(Op o)
{
    if (o.kind == BCAST || o.kind == ALLGATHER) o.seq = o.comm->seq++;
    t_ops.push_back(o);
    if (t_depth > 0) return ncclSuccess;
    std::vector<Op> ops;
    ops.swap(t_ops);
    return run_group(ops);
}

}  // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId *id)
{
    std::random_device rd;
    memset(id, 0, sizeof(*id));
    for (int i = 0; i < 16; i++) id->internal[i] = (char)(rd() & 0xff);
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t *comm, int nranks, ncclUniqueId id, int rank)
{
    if (rank < 0 || rank >= nranks) return ncclInvalidArgument;
    std::string key(id.internal, id.internal + 16);
    World *w;
    {
        std::lock_guard<std::mutex> lk(g_mu);
        auto it = g_worlds.find(key);
        if (it == g_worlds.end()) it = g_worlds.emplace(key, new World(nranks)).first;
        w = it->second;
    }
    if (w->n != nranks) return ncclInvalidArgument;
    ncclComm *c = new ncclComm();
    c->w = w; c->rank = rank; c->n = nranks;
    // CommInitRank is collective: wait for every rank
    std::unique_lock<std::mutex> lk(w->mu);
    w->joined[rank] = true;
    w->cv.notify_all();
    w->cv.wait(lk, [&] { for (bool j : w->joined) if (!j) return false; return true; });
    *comm = c;
    return ncclSuccess;
}

ncclResult_t ncclCommSplit(ncclComm_t comm, int color, int key, ncclComm_t *newcomm, ncclConfig_t *)
{
    World *w = comm->w;
    const long seq = comm->seq++;
    std::unique_lock<std::mutex> lk(w->mu);
    Coll &c = w->coll[seq];
    if (c.color.empty()) { c.color.assign(w->n, -2); c.key.assign(w->n, 0); }
    c.color[comm->rank] = color;
    c.key[comm->rank] = key;
    c.posted++;
    w->cv.notify_all();
    w->cv.wait(lk, [&] { return c.posted == w->n; });
    *newcomm = nullptr;
    if (color < 0) return ncclSuccess;
    std::vector<std::pair<int, int>> members;   // (key, parent rank)
    for (int r = 0; r < w->n; r++)
        if (c.color[r] == color) members.push_back({c.key[r], r});
    std::sort(members.begin(), members.end());
    World *&sw = c.split_worlds[color];
    if (!sw) sw = new World((int)members.size());
    int myrank = 0;
    for (size_t i = 0; i < members.size(); i++)
        if (members[i].second == comm->rank) myrank = (int)i;
    ncclComm *nc = new ncclComm();
    nc->w = sw; nc->rank = myrank; nc->n = (int)members.size();
    *newcomm = nc;
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm)
{
    delete comm;
    return ncclSuccess;
}

ncclResult_t ncclGroupStart()
{
    t_depth++;
    return ncclSuccess;
}

ncclResult_t ncclGroupEnd()
{
    if (t_depth <= 0) return ncclInvalidUsage;
    if (--t_depth > 0) return ncclSuccess;
    std::vector<Op> ops;
    ops.swap(t_ops);
    return run_group(ops);
}

ncclResult_t ncclSend(const void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t s)
{
    return submit(Op{SEND, buf, nullptr, count * dsize(t), peer, comm, s, 0, nullptr});
}

ncclResult_t ncclRecv(void *buf, size_t count, ncclDataType_t t, int peer, ncclComm_t comm, cudaStream_t s)
{
    return submit(Op{RECV, nullptr, buf, count * dsize(t), peer, comm, s, 0, nullptr});
}

ncclResult_t ncclBroadcast(const void *sbuf, void *rbuf, size_t count, ncclDataType_t t, int root, ncclComm_t comm,
                           cudaStream_t s)
{
    return submit(Op{BCAST, sbuf, rbuf, count * dsize(t), root, comm, s, 0, nullptr});
}

ncclResult_t ncclAllGather(const void *sbuf, void *rbuf, size_t count, ncclDataType_t t, ncclComm_t comm,
                           cudaStream_t s)
{
    return submit(Op{ALLGATHER, sbuf, rbuf, count * dsize(t), -1, comm, s, 0, nullptr});
}

const char *ncclGetErrorString(ncclResult_t r)
{
    return r == ncclSuccess ? "success (loopback)" : "error (loopback)";
}

}  // extern "C"
