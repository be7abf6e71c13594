// nccl_comm.cu -- see nccl_comm.hpp.  Collectives of the sharded path over NCCL (NVLink 5 / NVSwitch on a B200 box):
//   all-to-all-v   grouped ncclSend/ncclRecv of byte ranges (candidate keys, look-up requests/replies, halos)
//   all-reduce     ncclAllReduce (norms: 2-4 doubles; selection histograms: 2048 x u32)
//   host variants  the few-byte blocking collectives (counts, sizes, tie keys) staged through a small device buffer
// Two communicators: `main` for everything the context's stream orders, `halo` for the halo exchange, which runs on
// its own stream beside the interior rows of the SpMV.
#include "nccl_comm.hpp"

#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <stdexcept>
#include <vector>

namespace pb {

namespace {
struct Api {
    void* lib = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*AllReduce)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Send)(const void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*Recv)(void*, size_t, ncclDataType_t, int, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*GroupStart)() = nullptr;
    ncclResult_t (*GroupEnd)() = nullptr;
};

Api& api() {
    static Api a;
    if (a.lib) return a;
    const char* names[] = {"libnccl.so.2", "libnccl.so"};
    for (const char* nm : names) {
        a.lib = dlopen(nm, RTLD_NOW | RTLD_GLOBAL);
        if (a.lib) break;
    }
    if (!a.lib) throw std::runtime_error(std::string("NCCL transport: cannot load libnccl.so.2 (") + dlerror() + ")");
    auto sym = [&](const char* s) {
        void* p = dlsym(a.lib, s);
        if (!p) throw std::runtime_error(std::string("NCCL transport: symbol missing: ") + s);
        return p;
    };
    a.GetVersion = reinterpret_cast<decltype(a.GetVersion)>(sym("ncclGetVersion"));
    a.GetUniqueId = reinterpret_cast<decltype(a.GetUniqueId)>(sym("ncclGetUniqueId"));
    a.CommInitRank = reinterpret_cast<decltype(a.CommInitRank)>(sym("ncclCommInitRank"));
    a.CommDestroy = reinterpret_cast<decltype(a.CommDestroy)>(sym("ncclCommDestroy"));
    a.GetErrorString = reinterpret_cast<decltype(a.GetErrorString)>(sym("ncclGetErrorString"));
    a.AllReduce = reinterpret_cast<decltype(a.AllReduce)>(sym("ncclAllReduce"));
    a.AllGather = reinterpret_cast<decltype(a.AllGather)>(sym("ncclAllGather"));
    a.Send = reinterpret_cast<decltype(a.Send)>(sym("ncclSend"));
    a.Recv = reinterpret_cast<decltype(a.Recv)>(sym("ncclRecv"));
    a.GroupStart = reinterpret_cast<decltype(a.GroupStart)>(sym("ncclGroupStart"));
    a.GroupEnd = reinterpret_cast<decltype(a.GroupEnd)>(sym("ncclGroupEnd"));
    return a;
}

void nccl_ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw std::runtime_error(std::string("NCCL error in ") + what + ": " + api().GetErrorString(r));
}
void cuda_ok(cudaError_t e, const char* what) {
    if (e != cudaSuccess) throw std::runtime_error(std::string("CUDA error in ") + what + ": " + cudaGetErrorString(e));
}
}  // namespace

struct NcclTransport {
    int device = 0, rank = 0, world = 1, version = 0;
    ncclComm_t main = nullptr, halo = nullptr;
    cudaStream_t* stream = nullptr;  // the owning context's stream variable
    void* d_stage = nullptr;         // device staging of the host-side collectives
    size_t d_cap = 0;
    std::string err;
    uint64_t n_alltoallv = 0, n_allreduce = 0, n_host = 0;

    void* stage(size_t bytes) {
        if (bytes > d_cap) {
            if (d_stage) cudaFree(d_stage);
            d_cap = bytes + bytes / 2 + 4096;
            cuda_ok(cudaMalloc(&d_stage, d_cap), "cudaMalloc(staging)");
        }
        return d_stage;
    }
    template <class F>
    int guard(F&& f) {
        try {
            f();
            return 0;
        } catch (const std::exception& e) {
            err = e.what();
            std::fprintf(stderr, "[paces_b200 rank %d] %s\n", rank, err.c_str());
            return 1;
        }
    }
    /// in-place all-reduce of a small host array through the staging buffer
    void allreduce_host(void* buf, size_t n, size_t esize, ncclDataType_t dt) {
        void* d = stage(n * esize);
        cudaStream_t s = *stream;
        cuda_ok(cudaMemcpyAsync(d, buf, n * esize, cudaMemcpyHostToDevice, s), "H2D");
        nccl_ok(api().AllReduce(d, d, n, dt, ncclSum, main, s), "ncclAllReduce");
        cuda_ok(cudaMemcpyAsync(buf, d, n * esize, cudaMemcpyDeviceToHost, s), "D2H");
        cuda_ok(cudaStreamSynchronize(s), "synchronize");
        ++n_host;
    }
    void alltoallv(ncclComm_t comm, const void* send, const uint64_t* sc, void* recv, const uint64_t* rc, uint64_t eb,
                   cudaStream_t s) {
        const char* sp = static_cast<const char*>(send);
        char* rp = static_cast<char*>(recv);
        nccl_ok(api().GroupStart(), "ncclGroupStart");
        for (int p = 0; p < world; ++p) {
            if (sc[p]) nccl_ok(api().Send(sp, sc[p] * eb, ncclChar, p, comm, s), "ncclSend");
            if (rc[p]) nccl_ok(api().Recv(rp, rc[p] * eb, ncclChar, p, comm, s), "ncclRecv");
            sp += sc[p] * eb;
            rp += rc[p] * eb;
        }
        nccl_ok(api().GroupEnd(), "ncclGroupEnd");
        ++n_alltoallv;
    }
};

void nccl_make_unique_id(uint8_t* id) {
    ncclUniqueId a, b;
    nccl_ok(api().GetUniqueId(&a), "ncclGetUniqueId");
    nccl_ok(api().GetUniqueId(&b), "ncclGetUniqueId");
    std::memcpy(id, &a, sizeof(a));
    std::memcpy(id + sizeof(a), &b, sizeof(b));
}

NcclTransport* nccl_transport_create(int device, int rank, int world, const uint8_t* id, cudaStream_t* stream) {
    auto* t = new NcclTransport;
    t->device = device;
    t->rank = rank;
    t->world = world;
    t->stream = stream;
    try {
        cuda_ok(cudaSetDevice(device), "cudaSetDevice");
        api().GetVersion(&t->version);
        ncclUniqueId a, b;
        std::memcpy(&a, id, sizeof(a));
        std::memcpy(&b, id + sizeof(a), sizeof(b));
        nccl_ok(api().CommInitRank(&t->main, world, a, rank), "ncclCommInitRank(main)");
        nccl_ok(api().CommInitRank(&t->halo, world, b, rank), "ncclCommInitRank(halo)");
        t->stage(1 << 16);
    } catch (...) {
        nccl_transport_destroy(t);
        throw;
    }
    return t;
}

void nccl_transport_destroy(NcclTransport* t) {
    if (!t) return;
    cudaSetDevice(t->device);
    if (t->halo) api().CommDestroy(t->halo);
    if (t->main) api().CommDestroy(t->main);
    if (t->d_stage) cudaFree(t->d_stage);
    delete t;
}

std::string nccl_transport_describe(const NcclTransport* t) {
    return "NCCL " + std::to_string(t->version) + ", rank " + std::to_string(t->rank) + "/" + std::to_string(t->world) +
           ", alltoallv " + std::to_string(t->n_alltoallv) + ", allreduce " + std::to_string(t->n_allreduce) +
           ", host collectives " + std::to_string(t->n_host);
}

namespace {
NcclTransport* T(void* user) { return static_cast<NcclTransport*>(user); }

int cb_allreduce_f64_host(void* u, double* buf, uint64_t n) {
    return T(u)->guard([&] { T(u)->allreduce_host(buf, n, 8, ncclDouble); });
}
int cb_allreduce_u64_host(void* u, uint64_t* buf, uint64_t n) {
    return T(u)->guard([&] { T(u)->allreduce_host(buf, n, 8, ncclUint64); });
}
int cb_alltoall_u64_host(void* u, const uint64_t* send, uint64_t* recv) {
    NcclTransport* t = T(u);
    return t->guard([&] {
        const size_t P = size_t(t->world);
        char* d = static_cast<char*>(t->stage(2 * P * 8));
        cudaStream_t s = *t->stream;
        cuda_ok(cudaMemcpyAsync(d, send, P * 8, cudaMemcpyHostToDevice, s), "H2D");
        std::vector<uint64_t> ones(P, 1);
        t->alltoallv(t->main, d, ones.data(), d + P * 8, ones.data(), 8, s);
        cuda_ok(cudaMemcpyAsync(recv, d + P * 8, P * 8, cudaMemcpyDeviceToHost, s), "D2H");
        cuda_ok(cudaStreamSynchronize(s), "synchronize");
        ++t->n_host;
    });
}
int cb_allgather_host(void* u, const void* send, uint64_t nbytes, void* recv) {
    NcclTransport* t = T(u);
    return t->guard([&] {
        const size_t P = size_t(t->world);
        if (nbytes == 0) return;
        char* d = static_cast<char*>(t->stage((P + 1) * nbytes));
        cudaStream_t s = *t->stream;
        cuda_ok(cudaMemcpyAsync(d, send, nbytes, cudaMemcpyHostToDevice, s), "H2D");
        nccl_ok(api().AllGather(d, d + nbytes, nbytes, ncclChar, t->main, s), "ncclAllGather");
        cuda_ok(cudaMemcpyAsync(recv, d + nbytes, P * nbytes, cudaMemcpyDeviceToHost, s), "D2H");
        cuda_ok(cudaStreamSynchronize(s), "synchronize");
        ++t->n_host;
    });
}
int cb_alltoallv_dev(void* u, const void* send, const uint64_t* sc, void* recv, const uint64_t* rc, uint64_t eb,
                     void* stream) {
    NcclTransport* t = T(u);
    return t->guard([&] { t->alltoallv(t->main, send, sc, recv, rc, eb, static_cast<cudaStream_t>(stream)); });
}
int cb_alltoallv_dev2(void* u, const void* send, const uint64_t* sc, void* recv, const uint64_t* rc, uint64_t eb,
                      void* stream) {
    NcclTransport* t = T(u);
    return t->guard([&] { t->alltoallv(t->halo, send, sc, recv, rc, eb, static_cast<cudaStream_t>(stream)); });
}
int cb_allreduce_f64_dev(void* u, double* buf, uint64_t n, void* stream) {
    NcclTransport* t = T(u);
    return t->guard([&] {
        nccl_ok(api().AllReduce(buf, buf, n, ncclDouble, ncclSum, t->main, static_cast<cudaStream_t>(stream)),
                "ncclAllReduce(f64)");
        ++t->n_allreduce;
    });
}
int cb_allreduce_u32_dev(void* u, uint32_t* buf, uint64_t n, void* stream) {
    NcclTransport* t = T(u);
    return t->guard([&] {
        nccl_ok(api().AllReduce(buf, buf, n, ncclUint32, ncclSum, t->main, static_cast<cudaStream_t>(stream)),
                "ncclAllReduce(u32)");
        ++t->n_allreduce;
    });
}
}  // namespace

pb200_comm_ops nccl_transport_ops(NcclTransport* t) {
    pb200_comm_ops o{};
    o.user = t;
    o.allreduce_f64_host = cb_allreduce_f64_host;
    o.allreduce_u64_host = cb_allreduce_u64_host;
    o.alltoall_u64_host = cb_alltoall_u64_host;
    o.allgather_host = cb_allgather_host;
    o.alltoallv_dev = cb_alltoallv_dev;
    o.allreduce_f64_dev = cb_allreduce_f64_dev;
    o.allreduce_u32_dev = cb_allreduce_u32_dev;
    o.alltoallv_dev2 = cb_alltoallv_dev2;
    return o;
}

}  // namespace pb
