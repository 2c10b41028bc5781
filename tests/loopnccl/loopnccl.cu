// In-process loopback NCCL for multi-rank tests on ONE GPU (test
// infrastructure only; the product loads it solely when ACO_NCCL_LIB points
// here).  Real NCCL refuses two ranks on one device ("Duplicate GPU
// detected"), so the engine's world > 1 protocol — communicator init, the
// statistics all-reduces, the delta all-reduce on every wire, the row-sharded
// gather's send/recv + all-gather, the nn slot/record exchange, the multicast
// setup's agreement — could not run anywhere but an 8-GPU node.  Here every
// rank is a thread of one process with its own engine context on device 0:
//
//   * a communicator is a shared object keyed by the unique id; init blocks
//     until all ranks joined (NCCL's init is collective too);
//   * every call outside ncclGroupStart/End is a group of one; a rank posts
//     its k-th group with an event on its stream; the last rank to post group
//     k executes it on a private stream after waiting on every rank's event
//     (collectives in call order, the i-th send a->b matched with the i-th
//     recv on b from a), records a completion event, and every rank's stream
//     waits on it before its call returns;
//   * reductions run in rank order (deterministic; real NCCL's order differs,
//     which the engine's tolerances already allow for).
//
// Build: nvcc -O2 -std=c++17 -shared -Xcompiler -fPIC loopnccl.cu -o libloopnccl.so
#include <cuda_runtime.h>
#include <nccl.h>

#include <condition_variable>
#include <cstdint>
#include <cstring>
#include <deque>
#include <map>
#include <memory>
#include <mutex>
#include <random>
#include <string>
#include <vector>

namespace {

enum Kind { ALLREDUCE, ALLGATHER, BROADCAST, SEND, RECV };

struct Op {
    Kind kind;
    const void* send;
    void* recv;
    size_t count;
    ncclDataType_t dt;
    ncclRedOp_t op;
    int peer; // SEND/RECV peer, BROADCAST root
};

struct Posted {
    std::vector<Op> ops;
    cudaEvent_t ready;
    cudaStream_t stream;
};

struct Shared {
    std::mutex mu;
    std::condition_variable cv;
    int nranks = 0, joined = 0, alive = 0;
    std::vector<std::deque<Posted>> posted; // [rank] groups not yet executed
    std::vector<long> npost;                // groups posted per rank
    long executed = 0;                      // groups executed
    std::map<long, cudaEvent_t> done;       // group -> completion event
    cudaStream_t cs = nullptr;
    void* tmp = nullptr;
    size_t tmp_bytes = 0;
};

struct Registry {
    std::mutex mu;
    std::map<std::string, std::shared_ptr<Shared>> comms;
};
Registry& reg() {
    static Registry r;
    return r;
}

size_t dt_size(ncclDataType_t t) {
    switch (t) {
    case ncclInt8: case ncclUint8: return 1;
    case ncclFloat16: case ncclBfloat16: return 2;
    case ncclInt32: case ncclUint32: case ncclFloat32: return 4;
    default: return 8;
    }
}

template <typename T>
__global__ void k_reduce(T* acc, const T* x, size_t n, int op) {
    for (size_t i = blockIdx.x * static_cast<size_t>(blockDim.x) + threadIdx.x; i < n;
         i += static_cast<size_t>(gridDim.x) * blockDim.x) {
        const T a = acc[i], b = x[i];
        acc[i] = op == ncclSum ? static_cast<T>(a + b) : op == ncclMin ? (b < a ? b : a) : (b > a ? b : a);
    }
}

template <typename T>
void reduce_t(void* acc, const void* x, size_t n, int op, cudaStream_t s) {
    const int grid = static_cast<int>(std::min<size_t>((n + 255) / 256, 4096));
    k_reduce<T><<<grid > 0 ? grid : 1, 256, 0, s>>>(static_cast<T*>(acc), static_cast<const T*>(x), n, op);
}

void reduce(void* acc, const void* x, size_t n, ncclDataType_t dt, int op, cudaStream_t s) {
    switch (dt) {
    case ncclInt32: reduce_t<int32_t>(acc, x, n, op, s); break;
    case ncclUint32: reduce_t<uint32_t>(acc, x, n, op, s); break;
    case ncclInt64: reduce_t<long long>(acc, x, n, op, s); break;
    case ncclUint64: reduce_t<unsigned long long>(acc, x, n, op, s); break;
    case ncclFloat32: reduce_t<float>(acc, x, n, op, s); break;
    case ncclFloat64: reduce_t<double>(acc, x, n, op, s); break;
    case ncclUint8: reduce_t<uint8_t>(acc, x, n, op, s); break;
    default: reduce_t<int8_t>(acc, x, n, op, s); break;
    }
}

// executes group k (every rank's group at the front of its queue); sh->mu held
void execute(Shared* sh) {
    const int R = sh->nranks;
    std::vector<Posted> g(R);
    for (int r = 0; r < R; ++r) {
        g[r] = sh->posted[r].front();
        sh->posted[r].pop_front();
        cudaStreamWaitEvent(sh->cs, g[r].ready, 0);
    }
    // collectives: the i-th collective of every rank belong together
    std::vector<std::vector<const Op*>> coll(R);
    for (int r = 0; r < R; ++r)
        for (const Op& o : g[r].ops)
            if (o.kind != SEND && o.kind != RECV) coll[r].push_back(&o);
    for (size_t i = 0; i < coll[0].size(); ++i) {
        const Op& o0 = *coll[0][i];
        const size_t bytes = o0.count * dt_size(o0.dt);
        if (o0.kind == ALLREDUCE) {
            if (sh->tmp_bytes < bytes) {
                if (sh->tmp) cudaFree(sh->tmp);
                cudaMalloc(&sh->tmp, bytes);
                sh->tmp_bytes = bytes;
            }
            cudaMemcpyAsync(sh->tmp, coll[0][i]->send, bytes, cudaMemcpyDeviceToDevice, sh->cs);
            for (int r = 1; r < R; ++r) reduce(sh->tmp, coll[r][i]->send, o0.count, o0.dt, o0.op, sh->cs);
            for (int r = 0; r < R; ++r)
                cudaMemcpyAsync(coll[r][i]->recv, sh->tmp, bytes, cudaMemcpyDeviceToDevice, sh->cs);
        } else if (o0.kind == ALLGATHER) {
            for (int r = 0; r < R; ++r)
                for (int q = 0; q < R; ++q) {
                    char* dst = static_cast<char*>(coll[r][i]->recv) + q * bytes;
                    if (dst != coll[q][i]->send)
                        cudaMemcpyAsync(dst, coll[q][i]->send, bytes, cudaMemcpyDeviceToDevice, sh->cs);
                }
        } else { // BROADCAST
            const int root = o0.peer;
            for (int r = 0; r < R; ++r)
                if (coll[r][i]->recv != coll[root][i]->send)
                    cudaMemcpyAsync(coll[r][i]->recv, coll[root][i]->send, bytes, cudaMemcpyDeviceToDevice,
                                    sh->cs);
        }
    }
    // point to point: the i-th send a->b with the i-th recv on b from a
    for (int a = 0; a < R; ++a) {
        std::map<int, int> nth; // peer -> sends seen
        for (const Op& o : g[a].ops) {
            if (o.kind != SEND) continue;
            const int b = o.peer, k = nth[b]++;
            int seen = 0;
            for (const Op& p : g[b].ops)
                if (p.kind == RECV && p.peer == a && seen++ == k) {
                    cudaMemcpyAsync(p.recv, o.send, o.count * dt_size(o.dt), cudaMemcpyDeviceToDevice, sh->cs);
                    break;
                }
        }
    }
    cudaEvent_t fin;
    cudaEventCreateWithFlags(&fin, cudaEventDisableTiming);
    cudaEventRecord(fin, sh->cs);
    sh->done[sh->executed] = fin;
    ++sh->executed;
    for (int r = 0; r < R; ++r) cudaEventDestroy(g[r].ready);
}

} // namespace

struct ncclComm {
    std::shared_ptr<Shared> sh;
    int rank;
};

namespace {
thread_local int g_depth = 0;
thread_local std::vector<Op> g_ops;
thread_local ncclComm_t g_comm = nullptr;
thread_local cudaStream_t g_stream = nullptr;

ncclResult_t post(ncclComm_t comm, cudaStream_t stream, std::vector<Op> ops) {
    Shared* sh = comm->sh.get();
    Posted p;
    p.ops = std::move(ops);
    p.stream = stream;
    cudaEventCreateWithFlags(&p.ready, cudaEventDisableTiming);
    cudaEventRecord(p.ready, stream);
    std::unique_lock<std::mutex> lk(sh->mu);
    const long k = sh->npost[comm->rank]++;
    sh->posted[comm->rank].push_back(p);
    bool all = true;
    for (int r = 0; r < sh->nranks; ++r) all = all && sh->npost[r] > k;
    if (all) {
        while (sh->executed <= k) execute(sh);
        sh->cv.notify_all();
    }
    sh->cv.wait(lk, [&] { return sh->executed > k; });
    cudaStreamWaitEvent(stream, sh->done[k], 0);
    return ncclSuccess;
}

ncclResult_t submit(ncclComm_t comm, cudaStream_t stream, const Op& op) {
    if (g_depth > 0) {
        g_ops.push_back(op);
        g_comm = comm;
        g_stream = stream;
        return ncclSuccess;
    }
    return post(comm, stream, {op});
}
} // namespace

extern "C" {

ncclResult_t ncclGetUniqueId(ncclUniqueId* id) {
    std::random_device rd;
    for (int i = 0; i < NCCL_UNIQUE_ID_BYTES; ++i) id->internal[i] = static_cast<char>(rd());
    return ncclSuccess;
}

ncclResult_t ncclCommInitRank(ncclComm_t* comm, int nranks, ncclUniqueId id, int rank) {
    std::shared_ptr<Shared> sh;
    {
        std::lock_guard<std::mutex> g(reg().mu);
        auto& slot = reg().comms[std::string(id.internal, NCCL_UNIQUE_ID_BYTES)];
        if (!slot) {
            slot = std::make_shared<Shared>();
            slot->nranks = nranks;
            slot->posted.resize(nranks);
            slot->npost.assign(nranks, 0);
            cudaStreamCreateWithFlags(&slot->cs, cudaStreamNonBlocking);
        }
        sh = slot;
    }
    if (rank < 0 || rank >= sh->nranks || nranks != sh->nranks) return ncclInvalidArgument;
    std::unique_lock<std::mutex> lk(sh->mu);
    ++sh->joined;
    ++sh->alive;
    sh->cv.notify_all();
    sh->cv.wait(lk, [&] { return sh->joined == sh->nranks; });
    *comm = new ncclComm{sh, rank};
    return ncclSuccess;
}

ncclResult_t ncclCommDestroy(ncclComm_t comm) {
    if (!comm) return ncclSuccess;
    {
        std::lock_guard<std::mutex> g(comm->sh->mu);
        --comm->sh->alive;
    }
    delete comm;
    return ncclSuccess;
}

ncclResult_t ncclAllReduce(const void* s, void* r, size_t count, ncclDataType_t dt, ncclRedOp_t op, ncclComm_t comm,
                           cudaStream_t stream) {
    return submit(comm, stream, Op{ALLREDUCE, s, r, count, dt, op, 0});
}
ncclResult_t ncclAllGather(const void* s, void* r, size_t count, ncclDataType_t dt, ncclComm_t comm,
                           cudaStream_t stream) {
    return submit(comm, stream, Op{ALLGATHER, s, r, count, dt, ncclSum, 0});
}
ncclResult_t ncclBroadcast(const void* s, void* r, size_t count, ncclDataType_t dt, int root, ncclComm_t comm,
                           cudaStream_t stream) {
    return submit(comm, stream, Op{BROADCAST, s, r, count, dt, ncclSum, root});
}
ncclResult_t ncclSend(const void* s, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm,
                      cudaStream_t stream) {
    return submit(comm, stream, Op{SEND, s, nullptr, count, dt, ncclSum, peer});
}
ncclResult_t ncclRecv(void* r, size_t count, ncclDataType_t dt, int peer, ncclComm_t comm, cudaStream_t stream) {
    return submit(comm, stream, Op{RECV, nullptr, r, count, dt, ncclSum, peer});
}
ncclResult_t ncclGroupStart() {
    ++g_depth;
    return ncclSuccess;
}
ncclResult_t ncclGroupEnd() {
    if (--g_depth > 0) return ncclSuccess;
    if (g_ops.empty()) return ncclSuccess;
    std::vector<Op> ops;
    ops.swap(g_ops);
    return post(g_comm, g_stream, std::move(ops));
}
const char* ncclGetErrorString(ncclResult_t) { return "loopnccl error"; }

} // extern "C"
