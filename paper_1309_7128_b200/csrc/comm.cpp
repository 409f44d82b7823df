// comm.cpp — multi-GPU communicator for the strip decomposition.
//
// One process per GPU; the ranks share an NCCL communicator created from a
// 128-byte ncclUniqueId (rank 0 makes it with ismg_nccl_unique_id and hands it
// to the others through the caller's own channel, e.g. torch.distributed).
// Fine rows are split into strips of whole coarse tiles (strip_rows), so every
// coarse cell, and therefore every tile sum, belongs to one rank.
#include <nccl.h>

#include <algorithm>
#include <cstring>
#include <string>
#include <utility>

#include "engine.h"

namespace ismgb {

Comm* make_comm(int device, const void* unique_id, int rank, int nranks) {
    if (nranks < 1 || rank < 0 || rank >= nranks) fail(ISMG_ERR_INVALID_ARGUMENT, "comm: bad rank / nranks");
    auto* c = new Comm();
    c->rank = rank, c->nranks = nranks;
    ISMG_CUDA(cudaSetDevice(device));
    ncclUniqueId id;
    static_assert(sizeof(id) == 128, "ncclUniqueId is 128 bytes");
    std::memcpy(&id, unique_id, sizeof(id));
    const ncclResult_t r = ncclCommInitRank(reinterpret_cast<ncclComm_t*>(&c->nccl), nranks, id, rank);
    if (r != ncclSuccess) {
        delete c;
        fail(ISMG_ERR_NCCL, std::string("ncclCommInitRank: ") + ncclGetErrorString(r));
    }
    return c;
}

void destroy_comm(Comm* c) {
    if (!c) return;
    if (c->nccl) ncclCommDestroy(reinterpret_cast<ncclComm_t>(c->nccl));
    delete c;
}

void nccl_unique_id(void* out) {
    ncclUniqueId id;
    const ncclResult_t r = ncclGetUniqueId(&id);
    if (r != ncclSuccess) fail(ISMG_ERR_NCCL, std::string("ncclGetUniqueId: ") + ncclGetErrorString(r));
    std::memcpy(out, &id, sizeof(id));
}

// Rows [r0, r1) of rank `rank`: whole tiles, as even as possible (the first
// ntiles % nranks ranks take one tile more). Host-only; no device needed.
void strip_rows(int ny, int tile, int nranks, int rank, int* r0, int* r1) {
    if (ny < 1 || tile < 1 || nranks < 1 || rank < 0 || rank >= nranks)
        fail(ISMG_ERR_INVALID_ARGUMENT, "strip_rows: bad arguments");
    strip_of(ny, tile, nranks, rank, r0, r1);
}

static ncclComm_t C(const Comm& c) { return reinterpret_cast<ncclComm_t>(c.nccl); }
static void ok(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) fail(ISMG_ERR_NCCL, std::string(what) + ": " + ncclGetErrorString(r));
}

// MAX over [0, nmax) and SUM over [nmax, nmax + nsum) of a device vector (in place)
void comm_reduce_scalars(Comm& c, double* v, int nmax, int nsum, cudaStream_t st) {
    ok(ncclGroupStart(), "ncclGroupStart");
    ok(ncclAllReduce(v, v, size_t(nmax), ncclDouble, ncclMax, C(c), st), "ncclAllReduce(max)");
    ok(ncclAllReduce(v + nmax, v + nmax, size_t(nsum), ncclDouble, ncclSum, C(c), st), "ncclAllReduce(sum)");
    ok(ncclGroupEnd(), "ncclGroupEnd");
}

// Every rank's rows [rows_of(r)) of a pitched buffer (origin-based) to every rank,
// in place: one broadcast per rank, rooted at the owner.
void comm_gather_rows(Comm& c, double* origin, int64_t pitch, const std::vector<std::pair<int, int>>& rows,
                      cudaStream_t st) {
    ok(ncclGroupStart(), "ncclGroupStart");
    for (int r = 0; r < c.nranks; ++r) {
        const int a = rows[size_t(r)].first, b = rows[size_t(r)].second;
        if (b <= a) continue;
        double* p = origin + int64_t(a) * pitch;
        const size_t count = size_t(int64_t(b - a) * pitch);
        ok(ncclBroadcast(p, p, count, ncclDouble, r, C(c), st), "ncclBroadcast");
    }
    ok(ncclGroupEnd(), "ncclGroupEnd");
}

// Every rank's pack of `count` doubles to every rank (one NCCL call per fine pass).
void comm_allgather(Comm& c, const double* pack, double* gathered, size_t count, cudaStream_t st) {
    ok(ncclAllGather(pack, gathered, count, ncclDouble, C(c), st), "ncclAllGather");
}

// Halo rows: send[0] -> rank-1's recv[1], send[1] -> rank+1's recv[0] (count doubles each).
void comm_halo(Comm& c, double* const send[2], double* const recv[2], size_t count, cudaStream_t st) {
    ok(ncclGroupStart(), "ncclGroupStart");
    if (c.rank > 0) {
        ok(ncclSend(send[0], count, ncclDouble, c.rank - 1, C(c), st), "ncclSend");
        ok(ncclRecv(recv[0], count, ncclDouble, c.rank - 1, C(c), st), "ncclRecv");
    }
    if (c.rank + 1 < c.nranks) {
        ok(ncclSend(send[1], count, ncclDouble, c.rank + 1, C(c), st), "ncclSend");
        ok(ncclRecv(recv[1], count, ncclDouble, c.rank + 1, C(c), st), "ncclRecv");
    }
    ok(ncclGroupEnd(), "ncclGroupEnd");
}

}  // namespace ismgb
