// The library's own NCCL communicator and the two collectives of the path:
//   N1 — broadcast of the k x d centroids from rank 0 (a1 runs on rank 0 only);
//   N2 — the merge-record exchange, per peer ncclSend / ncclRecv in one group.
// One rank per GPU; the caller bootstraps the communicator by sharing the 128-byte unique id of
// rank 0 (any out-of-band channel: a file, MPI, torch.distributed).
#include <nccl.h>

#include "common.cuh"

namespace sg {

struct Comm {
    ncclComm_t nccl = nullptr;
    int rank = 0, world = 1;
};

static sg_status nccl_status(ncclResult_t r, const char* what) {
    set_error("NCCL error %s (%d) in %s", ncclGetErrorString(r), (int)r, what);
    return SG_ERR_NCCL;
}

#define SG_NCCL(call)                                              \
    do {                                                           \
        ncclResult_t _r = (call);                                  \
        if (_r != ncclSuccess) return sg::nccl_status(_r, #call);  \
    } while (0)

sg_status comm_rank_world(void* comm, int* rank, int* world) {
    if (!comm) { *rank = 0; *world = 1; return SG_OK; }
    const Comm* c = (const Comm*)comm;
    *rank = c->rank;
    *world = c->world;
    return SG_OK;
}

sg_status exchange_records_run(void* comm, const uint32_t* sendbuf, const uint64_t* send_host, uint32_t* recvbuf,
                               const uint64_t* recv_host, uint32_t words, cudaStream_t st) {
    if (!comm) return SG_OK;   // world 1: nothing leaves the rank
    const Comm* c = (const Comm*)comm;
    uint64_t so = 0, ro = 0;
    SG_NCCL(ncclGroupStart());
    for (int p = 0; p < c->world; p++) {
        const size_t ns = (size_t)send_host[p] * words, nr = (size_t)recv_host[p] * words;
        if (p != c->rank) {
            if (ns) SG_NCCL(ncclSend(sendbuf + so, ns, ncclUint32, p, c->nccl, st));
            if (nr) SG_NCCL(ncclRecv(recvbuf + ro, nr, ncclUint32, p, c->nccl, st));
        }
        so += ns;
        ro += nr;
    }
    SG_NCCL(ncclGroupEnd());
    return SG_OK;
}

}  // namespace sg

using namespace sg;

extern "C" {

sg_status scalegann_get_unique_id(uint8_t out[128]) {
    SG_CHECK_ARG(out, "get_unique_id: null out");
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    SG_NCCL(ncclGetUniqueId(&id));
    memcpy(out, &id, 128);
    return SG_OK;
}

sg_status scalegann_comm_init(int rank, int world, const uint8_t uid[128], void** comm) {
    SG_CHECK_ARG(uid && comm && world >= 1 && rank >= 0 && rank < world, "comm_init: bad arguments");
    Comm* c = new Comm();
    c->rank = rank;
    c->world = world;
    ncclUniqueId id;
    memcpy(&id, uid, 128);
    ncclResult_t r = ncclCommInitRank(&c->nccl, world, id, rank);
    if (r != ncclSuccess) {
        delete c;
        return nccl_status(r, "ncclCommInitRank");
    }
    *comm = c;
    return SG_OK;
}

sg_status scalegann_comm_destroy(void* comm) {
    if (!comm) return SG_OK;
    Comm* c = (Comm*)comm;
    ncclResult_t r = ncclCommDestroy(c->nccl);
    delete c;
    if (r != ncclSuccess) return nccl_status(r, "ncclCommDestroy");
    return SG_OK;
}

sg_status scalegann_comm_rank(void* comm, int* rank, int* world) {
    SG_CHECK_ARG(rank && world, "comm_rank: null output");
    return comm_rank_world(comm, rank, world);
}

sg_status scalegann_broadcast_centroids(void* comm, float* centroids, uint32_t k, uint32_t d, void* stream) {
    SG_CHECK_ARG(centroids && k >= 1 && d >= 1, "broadcast_centroids: bad arguments");
    if (!comm) return SG_OK;
    const Comm* c = (const Comm*)comm;
    SG_NCCL(ncclBroadcast(centroids, centroids, (size_t)k * d, ncclFloat32, 0, c->nccl, S(stream)));
    return SG_OK;
}

sg_status scalegann_exchange_records(void* comm, const uint32_t* sendbuf, const uint64_t* send_host, uint32_t* recvbuf,
                                     const uint64_t* recv_host, uint32_t words, void* stream) {
    SG_CHECK_ARG(send_host && recv_host && words >= 1, "exchange_records: bad arguments");
    return exchange_records_run(comm, sendbuf, send_host, recvbuf, recv_host, words, S(stream));
}

}  // extern "C"
