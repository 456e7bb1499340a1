// Multi-GPU plumbing of the z-slab training path, inside
// libtgcu: no PyTorch, no MPI.
//
// A tgcu_comm is one rank of a job of `nranks` processes (one per GPU).
// Bootstrap: rank 0 listens on addr:port, every other rank connects (star of
// TCP sockets). That star carries the host-side collectives (allgather,
// barrier, fixed-order host all-reduce, routed point-to-point). Backends of
// the step's device collectives:
//   TGCU_COMM_NCCL: NCCL (dlopen'ed libnccl.so.2; rank 0's ncclUniqueId goes
//     over the star) — the all-reduce of the step's 5 loss partials runs on
//     the step's stream, in place in device memory, and the halo fallback is
//     grouped ncclSend/ncclRecv: the whole slab step stays stream-ordered.
//   TGCU_COMM_HOST: the same collectives staged through host memory over the
//     star (tests; ranks sharing one device, where NCCL refuses duplicate
//     GPUs). Sums are formed in rank order, so every rank sees the same bits.
// Per step (tgcu_slab_train_step): tgcu_slab_step_begin -> all-reduce of the
// partials -> tgcu_slab_step_finish -> halo planes (none when the brick
// kernel stores them into the neighbours over peer memory: tgcu_slab_connect
// sets that up with CUDA IPC handles exchanged over the star).
#include <arpa/inet.h>
#include <dlfcn.h>
#include <netdb.h>
#include <netinet/in.h>
#include <netinet/tcp.h>
#include <sys/socket.h>
#include <unistd.h>

#include <chrono>
#include <cstring>
#include <string>
#include <thread>
#include <vector>

#include "tg_internal.h"

using namespace tgcu;

namespace {

// ---- the NCCL subset used, resolved at run time --------------------------------
typedef struct ncclComm* ncclComm_t;
typedef struct {
    char internal[128];
} ncclUniqueId;
typedef int ncclResult_t;
enum { ncclFloat32 = 7, ncclFloat64 = 9 };
enum { ncclSum = 0, ncclMax = 2, ncclMin = 3 };

struct Nccl {
    void* lib = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, int, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
};

Nccl& nccl() {
    static Nccl n;
    if (n.lib) return n;
    void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
    if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
    if (!h) throw Error(TGCU_ERR_CUDA, std::string("comm: cannot load libnccl.so.2: ") + dlerror());
    auto sym = [&](const char* name) {
        void* p = dlsym(h, name);
        if (!p) throw Error(TGCU_ERR_CUDA, std::string("comm: libnccl lacks ") + name);
        return p;
    };
    n.GetUniqueId = reinterpret_cast<decltype(n.GetUniqueId)>(sym("ncclGetUniqueId"));
    n.CommInitRank = reinterpret_cast<decltype(n.CommInitRank)>(sym("ncclCommInitRank"));
    n.CommDestroy = reinterpret_cast<decltype(n.CommDestroy)>(sym("ncclCommDestroy"));
    n.AllReduce = reinterpret_cast<decltype(n.AllReduce)>(sym("ncclAllReduce"));
    n.Send = reinterpret_cast<decltype(n.Send)>(sym("ncclSend"));
    n.Recv = reinterpret_cast<decltype(n.Recv)>(sym("ncclRecv"));
    n.GroupStart = reinterpret_cast<decltype(n.GroupStart)>(sym("ncclGroupStart"));
    n.GroupEnd = reinterpret_cast<decltype(n.GroupEnd)>(sym("ncclGroupEnd"));
    n.GetErrorString = reinterpret_cast<decltype(n.GetErrorString)>(sym("ncclGetErrorString"));
    n.lib = h;
    return n;
}

#define TGCU_NCCL(expr)                                                                                  \
    do {                                                                                                 \
        const ncclResult_t _r = (expr);                                                                  \
        if (_r != 0) throw Error(TGCU_ERR_CUDA, std::string(#expr ": ") + nccl().GetErrorString(_r)); \
    } while (0)

// ---- TCP star ------------------------------------------------------------------
void send_all(int fd, const void* p, size_t n) {
    const char* c = static_cast<const char*>(p);
    while (n) {
        const ssize_t k = ::send(fd, c, n, MSG_NOSIGNAL);
        if (k <= 0) throw Error(TGCU_ERR_CUDA, "comm: connection lost (send)");
        c += k;
        n -= (size_t)k;
    }
}
void recv_all(int fd, void* p, size_t n) {
    char* c = static_cast<char*>(p);
    while (n) {
        const ssize_t k = ::recv(fd, c, n, 0);
        if (k <= 0) throw Error(TGCU_ERR_CUDA, "comm: connection lost (recv)");
        c += k;
        n -= (size_t)k;
    }
}
void send_blob(int fd, const std::vector<char>& b) {
    const uint64_t n = b.size();
    send_all(fd, &n, 8);
    if (n) send_all(fd, b.data(), n);
}
std::vector<char> recv_blob(int fd) {
    uint64_t n = 0;
    recv_all(fd, &n, 8);
    std::vector<char> b(n);
    if (n) recv_all(fd, b.data(), n);
    return b;
}

void tune(int fd) {
    int one = 1;
    setsockopt(fd, IPPROTO_TCP, TCP_NODELAY, &one, sizeof(one));
}

}  // namespace

struct tgcu_comm {
    int rank = 0, nranks = 1, device = 0, backend = TGCU_COMM_HOST;
    std::vector<int> peers;  // rank 0: sockets of ranks 1..n-1 (index = rank); others: peers[0] = rank 0
    ncclComm_t nc = nullptr;

    // Host collectives over the star (every rank calls them in the same order).
    std::vector<char> allgather(const void* in, size_t bytes) {
        std::vector<char> all(bytes * nranks);
        std::memcpy(all.data() + bytes * rank, in, bytes);
        if (nranks == 1) return all;
        if (rank == 0) {
            for (int r = 1; r < nranks; ++r) recv_all(peers[r], all.data() + bytes * r, bytes);
            for (int r = 1; r < nranks; ++r) send_all(peers[r], all.data(), all.size());
        } else {
            send_all(peers[0], in, bytes);
            recv_all(peers[0], all.data(), all.size());
        }
        return all;
    }
    void barrier() {
        const char c = 1;
        allgather(&c, 1);
    }
    // op: 0 sum, 1 max, 2 min; reduced in rank order (identical on every rank)
    void allreduce_host(double* buf, int n, int op) {
        const std::vector<char> all = allgather(buf, sizeof(double) * n);
        const double* a = reinterpret_cast<const double*>(all.data());
        for (int i = 0; i < n; ++i) {
            double acc = a[i];
            for (int r = 1; r < nranks; ++r) {
                const double x = a[(size_t)r * n + i];
                acc = op == 0 ? acc + x : (op == 1 ? (x > acc ? x : acc) : (x < acc ? x : acc));
            }
            buf[i] = acc;
        }
    }
    // Routed point-to-point: each rank passes (dst, bytes) messages and
    // receives the ones addressed to it as (src, bytes), in source-rank order.
    struct Msg {
        int peer;
        std::vector<char> data;
    };
    std::vector<Msg> exchange(const std::vector<Msg>& out) {
        auto pack = [](const std::vector<Msg>& ms) {
            std::vector<char> b;
            for (const Msg& m : ms) {
                const int32_t p = m.peer;
                const uint64_t n = m.data.size();
                b.insert(b.end(), reinterpret_cast<const char*>(&p), reinterpret_cast<const char*>(&p) + 4);
                b.insert(b.end(), reinterpret_cast<const char*>(&n), reinterpret_cast<const char*>(&n) + 8);
                b.insert(b.end(), m.data.begin(), m.data.end());
            }
            return b;
        };
        auto unpack = [](const std::vector<char>& b) {
            std::vector<Msg> ms;
            size_t o = 0;
            while (o < b.size()) {
                int32_t p;
                uint64_t n;
                std::memcpy(&p, b.data() + o, 4);
                std::memcpy(&n, b.data() + o + 4, 8);
                o += 12;
                ms.push_back({p, std::vector<char>(b.begin() + o, b.begin() + o + n)});
                o += n;
            }
            return ms;
        };
        if (nranks == 1) return {};
        if (rank != 0) {
            send_blob(peers[0], pack(out));
            return unpack(recv_blob(peers[0]));
        }
        std::vector<std::vector<Msg>> from(nranks);
        from[0] = out;
        for (int r = 1; r < nranks; ++r) from[r] = unpack(recv_blob(peers[r]));
        std::vector<std::vector<Msg>> to(nranks);
        for (int src = 0; src < nranks; ++src)
            for (const Msg& m : from[src]) {
                if (m.peer < 0 || m.peer >= nranks) throw Error(TGCU_ERR_INVALID_ARGUMENT, "comm: bad peer rank");
                to[m.peer].push_back({src, m.data});
            }
        for (int r = 1; r < nranks; ++r) send_blob(peers[r], pack(to[r]));
        return to[0];
    }
};

namespace {

void connect_star(tgcu_comm& c, const char* addr, int port, double timeout_s) {
    if (c.nranks == 1) return;
    const auto t_end = std::chrono::steady_clock::now() + std::chrono::duration<double>(timeout_s);
    if (c.rank == 0) {
        const int ls = ::socket(AF_INET, SOCK_STREAM, 0);
        if (ls < 0) throw Error(TGCU_ERR_CUDA, "comm: socket failed");
        int one = 1;
        setsockopt(ls, SOL_SOCKET, SO_REUSEADDR, &one, sizeof(one));
        sockaddr_in sa{};
        sa.sin_family = AF_INET;
        sa.sin_port = htons((uint16_t)port);
        sa.sin_addr.s_addr = htonl(INADDR_ANY);
        if (::bind(ls, reinterpret_cast<sockaddr*>(&sa), sizeof(sa)) != 0 || ::listen(ls, 1024) != 0) {
            ::close(ls);
            throw Error(TGCU_ERR_CUDA, "comm: cannot listen on port " + std::to_string(port));
        }
        c.peers.assign(c.nranks, -1);
        for (int k = 1; k < c.nranks; ++k) {
            const int fd = ::accept(ls, nullptr, nullptr);
            if (fd < 0) {
                ::close(ls);
                throw Error(TGCU_ERR_CUDA, "comm: accept failed");
            }
            tune(fd);
            int32_t r = -1;
            recv_all(fd, &r, 4);
            if (r <= 0 || r >= c.nranks || c.peers[r] >= 0) {
                ::close(ls);
                throw Error(TGCU_ERR_CUDA, "comm: bad or duplicate rank " + std::to_string(r));
            }
            c.peers[r] = fd;
        }
        ::close(ls);
        return;
    }
    addrinfo hints{}, *res = nullptr;
    hints.ai_family = AF_INET;
    hints.ai_socktype = SOCK_STREAM;
    if (getaddrinfo(addr, std::to_string(port).c_str(), &hints, &res) != 0 || !res)
        throw Error(TGCU_ERR_CUDA, std::string("comm: cannot resolve ") + addr);
    int fd = -1;
    while (true) {
        fd = ::socket(AF_INET, SOCK_STREAM, 0);
        if (fd >= 0 && ::connect(fd, res->ai_addr, res->ai_addrlen) == 0) break;
        if (fd >= 0) ::close(fd);
        if (std::chrono::steady_clock::now() > t_end) {
            freeaddrinfo(res);
            throw Error(TGCU_ERR_CUDA, std::string("comm: cannot connect to rank 0 at ") + addr + ":" +
                                           std::to_string(port));
        }
        std::this_thread::sleep_for(std::chrono::milliseconds(20));
    }
    freeaddrinfo(res);
    tune(fd);
    const int32_t r = c.rank;
    send_all(fd, &r, 4);
    c.peers.assign(1, fd);
}

}  // namespace

int tgcu_comm_create(const char* addr, int port, int rank, int nranks, int device, int backend, tgcu_comm** out) {
    if (out) *out = nullptr;
    tgcu_comm* c = nullptr;
    const int rc = guard([&] {
        require(out != nullptr, "comm_create: NULL out");
        require(nranks >= 1 && rank >= 0 && rank < nranks, "comm_create: bad rank / nranks");
        require(backend == TGCU_COMM_NCCL || backend == TGCU_COMM_HOST, "comm_create: unknown backend");
        require(nranks == 1 || (addr != nullptr && port > 0 && port < 65536), "comm_create: bad address");
        c = new tgcu_comm();
        c->rank = rank;
        c->nranks = nranks;
        c->device = device;
        c->backend = backend;
        connect_star(*c, addr, port, 120.0);
        if (backend == TGCU_COMM_NCCL) {
            Nccl& n = nccl();
            ncclUniqueId id{};
            if (rank == 0) TGCU_NCCL(n.GetUniqueId(&id));
            const std::vector<char> all = c->allgather(&id, sizeof(id));
            std::memcpy(&id, all.data(), sizeof(id));  // rank 0's
            TGCU_CUDA(cudaSetDevice(device));
            TGCU_NCCL(n.CommInitRank(&c->nc, nranks, id, rank));
        }
    });
    if (rc != TGCU_OK) {
        if (c) {
            for (int fd : c->peers)
                if (fd >= 0) ::close(fd);
            delete c;
        }
        return rc;
    }
    *out = c;
    return TGCU_OK;
}

int tgcu_comm_destroy(tgcu_comm* c) {
    return guard([&] {
        if (!c) return;
        if (c->nc) nccl().CommDestroy(c->nc);
        for (int fd : c->peers)
            if (fd >= 0) ::close(fd);
        delete c;
    });
}

int tgcu_comm_info(const tgcu_comm* c, int* rank, int* nranks, int* backend) {
    return guard([&] {
        require(c != nullptr, "comm_info: NULL comm");
        if (rank) *rank = c->rank;
        if (nranks) *nranks = c->nranks;
        if (backend) *backend = c->backend;
    });
}

int tgcu_comm_barrier(tgcu_comm* c) {
    return guard([&] {
        require(c != nullptr, "comm_barrier: NULL comm");
        c->barrier();
    });
}

int tgcu_comm_allreduce_host(tgcu_comm* c, double* buf, int n, int op) {
    return guard([&] {
        require(c != nullptr && (buf != nullptr || n == 0) && n >= 0 && op >= 0 && op <= 2,
                "comm_allreduce_host: bad argument");
        c->allreduce_host(buf, n, op);
    });
}

int tgcu_comm_allgather_host(tgcu_comm* c, const void* in, int64_t bytes, void* out) {
    return guard([&] {
        require(c != nullptr && in != nullptr && out != nullptr && bytes >= 0, "comm_allgather_host: bad argument");
        const std::vector<char> all = c->allgather(in, (size_t)bytes);
        std::memcpy(out, all.data(), all.size());
    });
}

int tgcu_comm_exchange_host(tgcu_comm* c, int nsend, const int* dst, const void* const* sbuf, const int64_t* sbytes,
                            int nrecv, const int* src, void* const* rbuf, const int64_t* rbytes) {
    return guard([&] {
        require(c != nullptr && nsend >= 0 && nrecv >= 0, "comm_exchange_host: bad argument");
        std::vector<tgcu_comm::Msg> out;
        for (int i = 0; i < nsend; ++i) {
            const char* b = static_cast<const char*>(sbuf[i]);
            out.push_back({dst[i], std::vector<char>(b, b + sbytes[i])});
        }
        const std::vector<tgcu_comm::Msg> in = c->exchange(out);
        std::vector<bool> used(in.size(), false);
        for (int j = 0; j < nrecv; ++j) {
            bool found = false;
            for (size_t k = 0; k < in.size() && !found; ++k) {
                if (used[k] || in[k].peer != src[j]) continue;
                require((int64_t)in[k].data.size() == rbytes[j], "comm_exchange_host: message size mismatch");
                std::memcpy(rbuf[j], in[k].data.data(), in[k].data.size());
                used[k] = found = true;
            }
            require(found, "comm_exchange_host: no message from rank " + std::to_string(src[j]));
        }
    });
}

// ---- slab training over a communicator -------------------------------------------

namespace {

void halo_exchange(tgcu_grid* h, tgcu_comm* c, cudaStream_t s) {
    float *s_lo, *s_hi, *r_lo, *r_hi;
    int64_t pf = 0;
    if (tgcu_slab_halo(h, &s_lo, &s_hi, &r_lo, &r_hi, &pf) != TGCU_OK) throw Error(TGCU_ERR_CUDA, tgcu_last_error());
    const int lo = c->rank - 1, hi = c->rank + 1;
    if (c->backend == TGCU_COMM_NCCL) {
        Nccl& n = nccl();
        TGCU_NCCL(n.GroupStart());
        if (s_lo) {
            TGCU_NCCL(n.Send(s_lo, (size_t)pf, ncclFloat32, lo, c->nc, s));
            TGCU_NCCL(n.Recv(r_lo, (size_t)pf, ncclFloat32, lo, c->nc, s));
        }
        if (s_hi) {
            TGCU_NCCL(n.Send(s_hi, (size_t)pf, ncclFloat32, hi, c->nc, s));
            TGCU_NCCL(n.Recv(r_hi, (size_t)pf, ncclFloat32, hi, c->nc, s));
        }
        TGCU_NCCL(n.GroupEnd());
        return;
    }
    std::vector<tgcu_comm::Msg> out;
    TGCU_CUDA(cudaStreamSynchronize(s));
    for (int side = 0; side < 2; ++side) {
        float* src = side == 0 ? s_lo : s_hi;
        if (!src) continue;
        tgcu_comm::Msg m{side == 0 ? lo : hi, std::vector<char>(sizeof(float) * pf)};
        TGCU_CUDA(cudaMemcpy(m.data.data(), src, m.data.size(), cudaMemcpyDeviceToHost));
        out.push_back(std::move(m));
    }
    for (const tgcu_comm::Msg& m : c->exchange(out)) {
        float* dst = m.peer == lo ? r_lo : (m.peer == hi ? r_hi : nullptr);
        require(dst != nullptr && m.data.size() == sizeof(float) * pf, "comm: unexpected halo message");
        TGCU_CUDA(cudaMemcpyAsync(dst, m.data.data(), m.data.size(), cudaMemcpyHostToDevice, s));
    }
    TGCU_CUDA(cudaStreamSynchronize(s));
}

}  // namespace

int tgcu_slab_connect(tgcu_grid* h, tgcu_comm* c, int fused_halo, int* fused_out) {
    return guard([&] {
        require(h != nullptr && c != nullptr, "slab_connect: NULL argument");
        Grid& g = h->g;
        require(g.slab, "slab_connect: not a slab grid");
        TGCU_CUDA(cudaSetDevice(g.device));
        int zb[5];
        if (tgcu_slab_info(h, &zb[0], &zb[1], &zb[2], &zb[3], &zb[4]) != TGCU_OK)
            throw Error(TGCU_ERR_CUDA, tgcu_last_error());
        // the ranks' slabs must tile the brick layers in rank order
        int lohi[2] = {g.zb0, g.zb0 + g.nb[2]};
        const std::vector<char> all = c->allgather(lohi, sizeof(lohi));
        const int* a = reinterpret_cast<const int*>(all.data());
        for (int r = 0; r < c->nranks; ++r) {
            const int want_lo = r == 0 ? 0 : a[2 * (r - 1) + 1];
            require(a[2 * r] == want_lo && a[2 * r + 1] > a[2 * r], "slab_connect: rank " + std::to_string(r) +
                                                                        " does not hold the next brick layers");
        }
        require(a[2 * (c->nranks - 1) + 1] == g.zb_global, "slab_connect: the slabs do not cover the grid");
        h->comm = c;
        // halo planes of the initial parameters
        halo_exchange(h, c, nullptr);
        TGCU_CUDA(cudaDeviceSynchronize());
        c->barrier();
        // fused halo: IPC handles of both parameter slots over the star, a probe round trip
        bool ok = fused_halo != 0 && c->nranks > 1;
        unsigned char blob[144] = {0};
        if (ok && tgcu_slab_ipc_export(h, blob) != TGCU_OK) ok = false;
        double okd = ok ? 1.0 : 0.0;
        c->allreduce_host(&okd, 1, 2);
        ok = okd > 0.0;
        if (ok) {
            const std::vector<char> blobs = c->allgather(blob, sizeof(blob));
            bool mine = true;
            if (c->rank > 0 && tgcu_slab_ipc_import(h, 0, blobs.data() + 144 * (c->rank - 1)) != TGCU_OK) mine = false;
            if (c->rank < c->nranks - 1 && tgcu_slab_ipc_import(h, 1, blobs.data() + 144 * (c->rank + 1)) != TGCU_OK)
                mine = false;
            okd = mine ? 1.0 : 0.0;
            c->allreduce_host(&okd, 1, 2);
            ok = okd > 0.0;
        }
        if (ok) {
            int pr = 1;
            if (tgcu_slab_peer_probe(h, 0, &pr) != TGCU_OK) pr = 0;
            c->barrier();
            int pr1 = 0;
            if (pr && tgcu_slab_peer_probe(h, 1, &pr1) != TGCU_OK) pr1 = 0;
            okd = (pr && pr1) ? 1.0 : 0.0;
            c->allreduce_host(&okd, 1, 2);
            ok = okd > 0.0;
        }
        if (!ok) {
            float* none[2] = {nullptr, nullptr};
            tgcu_slab_set_peer_planes(h, none, none);
        }
        h->fused_halo = ok;
        if (fused_out) *fused_out = ok ? 1 : 0;
        c->barrier();
    });
}

int tgcu_slab_train_step(tgcu_grid* h, const float* samples, int64_t n, int64_t n_global,
                         const tgcu_loss_config* cfg, tgcu_loss_terms* out, int flags, void* stream) {
    return guard([&] {
        require(h != nullptr && h->comm != nullptr, "slab_train_step: grid not connected (tgcu_slab_connect)");
        tgcu_comm* c = h->comm;
        cudaStream_t s = as_stream(stream);
        double* part = nullptr;
        if (tgcu_slab_step_begin(h, samples, n, n_global, cfg, &part, flags & ~TGCU_ASYNC, stream) != TGCU_OK)
            throw Error(TGCU_ERR_INVALID_ARGUMENT, tgcu_last_error());
        // profiled steps (tgcu_profile_begin): events around the collective phase
        const bool prof = h->g.prof_on && h->g.prof_this;
        auto mark = [&]() {
            if (h->coll_used >= h->coll_ev.size()) {
                cudaEvent_t e;
                TGCU_CUDA(cudaEventCreate(&e));
                h->coll_ev.push_back(e);
            }
            TGCU_CUDA(cudaEventRecord(h->coll_ev[h->coll_used++], s));
        };
        if (prof) mark();
        if (c->backend == TGCU_COMM_NCCL) {
            // in place on the step's stream: the finalize of every rank sees the same sums
            TGCU_NCCL(nccl().AllReduce(part, part, 5, ncclFloat64, ncclSum, c->nc, s));
        } else {
            double hp[5];
            TGCU_CUDA(cudaMemcpyAsync(hp, part, sizeof(hp), cudaMemcpyDeviceToHost, s));
            TGCU_CUDA(cudaStreamSynchronize(s));
            c->allreduce_host(hp, 5, 0);
            TGCU_CUDA(cudaMemcpyAsync(part, hp, sizeof(hp), cudaMemcpyHostToDevice, s));
        }
        if (prof) mark();  // (the finalize between the two phases is not counted)
        const int rc = tgcu_slab_step_finish(h, part, out, flags, stream);
        const std::string msg = rc == TGCU_OK ? std::string() : tgcu_last_error();
        // halo planes of the new parameters (the fused halo already stored them);
        // every rank reaches this point with the same commit decision
        if (prof) mark();
        if (!h->fused_halo) halo_exchange(h, c, s);
        if (prof) mark();
        if (rc != TGCU_OK) throw Error(rc, msg);
    });
}

int tgcu_slab_comm_profile(tgcu_grid* h, double* allreduce_ms, double* halo_ms, int* steps) {
    return guard([&] {
        require(h != nullptr, "slab_comm_profile: NULL grid");
        double ar = 0.0, hx = 0.0;
        const size_t n = h->coll_used / 4;
        for (size_t i = 0; i < n; ++i) {
            float a = 0.f, b = 0.f;
            TGCU_CUDA(cudaEventSynchronize(h->coll_ev[4 * i + 3]));
            TGCU_CUDA(cudaEventElapsedTime(&a, h->coll_ev[4 * i], h->coll_ev[4 * i + 1]));
            TGCU_CUDA(cudaEventElapsedTime(&b, h->coll_ev[4 * i + 2], h->coll_ev[4 * i + 3]));
            ar += a;
            hx += b;
        }
        if (allreduce_ms) *allreduce_ms = ar;
        if (halo_ms) *halo_ms = hx;
        if (steps) *steps = (int)n;
        h->coll_used = 0;
    });
}
