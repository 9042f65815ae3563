// nccl.cpp -- the one collective of the path: the validation checksum
// reduction across the per-GPU blocks of a partitioned vector (SURVEY.md
// section 8e).  The timed STREAM loop uses no collective: every block is
// processed by its owning GPU only.
//
// libnccl.so.2 is resolved with dlopen at first use, so the kernel library
// loads (and its symbols can be checked) on machines without NCCL, and a
// process that already loaded torch's NCCL reuses that copy.
#include "common.h"

#include <nccl.h>

#include <dlfcn.h>

#include <cstring>
#include <mutex>
#include <string>
#include <vector>

namespace {

struct nccl_api
{
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, int const*) = nullptr;
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_reduce)(void const*, void*, size_t, ncclDataType_t,
        ncclRedOp_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    char const* (*error_string)(ncclResult_t) = nullptr;
    bool ok = false;
    std::string why;
};

nccl_api const& api()
{
    static nccl_api a;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
            h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h)
        {
            char const* e = dlerror();
            a.why = std::string("dlopen libnccl.so.2 failed: ") + (e ? e : "?");
            return;
        }
        auto sym = [&](char const* name) { return dlsym(h, name); };
        a.comm_init_all = reinterpret_cast<decltype(a.comm_init_all)>(sym("ncclCommInitAll"));
        a.comm_destroy = reinterpret_cast<decltype(a.comm_destroy)>(sym("ncclCommDestroy"));
        a.get_unique_id = reinterpret_cast<decltype(a.get_unique_id)>(sym("ncclGetUniqueId"));
        a.comm_init_rank = reinterpret_cast<decltype(a.comm_init_rank)>(sym("ncclCommInitRank"));
        a.all_reduce = reinterpret_cast<decltype(a.all_reduce)>(sym("ncclAllReduce"));
        a.group_start = reinterpret_cast<decltype(a.group_start)>(sym("ncclGroupStart"));
        a.group_end = reinterpret_cast<decltype(a.group_end)>(sym("ncclGroupEnd"));
        a.error_string = reinterpret_cast<decltype(a.error_string)>(sym("ncclGetErrorString"));
        a.ok = a.comm_init_all && a.comm_destroy && a.all_reduce && a.group_start &&
            a.get_unique_id && a.comm_init_rank &&
            a.group_end && a.error_string;
        if (!a.ok)
            a.why = "libnccl.so.2 lacks required symbols";
    });
    return a;
}

int nccl_fail(ncclResult_t r, char const* what)
{
    auto const& a = api();
    return coloc_cuda::fail(COLOC_ERR_NCCL,
        std::string(what) + ": " + (a.error_string ? a.error_string(r) : "nccl error"));
}

}    // namespace

extern "C" {

int coloc_cuda_nccl_init_all(int ndev, const int* devs, void** comms_out)
{
    if (ndev <= 0 || !devs || !comms_out)
        return coloc_cuda::fail(COLOC_ERR_INVALID_ARGUMENT, "nccl_init_all: bad arguments");
    auto const& a = api();
    if (!a.ok)
        return coloc_cuda::fail(COLOC_ERR_NCCL, a.why);
    std::vector<ncclComm_t> comms(std::size_t(ndev), nullptr);
    ncclResult_t r = a.comm_init_all(comms.data(), ndev, devs);
    if (r != ncclSuccess)
        return nccl_fail(r, "ncclCommInitAll");
    for (int i = 0; i < ndev; ++i)
        comms_out[i] = comms[std::size_t(i)];
    return COLOC_OK;
}

int coloc_cuda_nccl_allreduce_sum_f64(int ndev, void* const* comms,
    double* const* bufs, size_t count, void* const* streams)
{
    if (ndev <= 0 || !comms || !bufs || !streams)
        return coloc_cuda::fail(COLOC_ERR_INVALID_ARGUMENT, "nccl_allreduce: bad arguments");
    auto const& a = api();
    if (!a.ok)
        return coloc_cuda::fail(COLOC_ERR_NCCL, a.why);
    ncclResult_t r = a.group_start();
    if (r != ncclSuccess)
        return nccl_fail(r, "ncclGroupStart");
    ncclResult_t first = ncclSuccess;
    for (int i = 0; i < ndev; ++i)
    {
        r = a.all_reduce(bufs[i], bufs[i], count, ncclFloat64, ncclSum,
            static_cast<ncclComm_t>(comms[i]), static_cast<cudaStream_t>(streams[i]));
        if (r != ncclSuccess && first == ncclSuccess)
            first = r;
    }
    r = a.group_end();
    if (first != ncclSuccess)
        return nccl_fail(first, "ncclAllReduce");
    if (r != ncclSuccess)
        return nccl_fail(r, "ncclGroupEnd");
    return COLOC_OK;
}

int coloc_cuda_nccl_unique_id(void* id_out, size_t bytes)
{
    if (!id_out || bytes < sizeof(ncclUniqueId))
        return coloc_cuda::fail(COLOC_ERR_INVALID_ARGUMENT,
            "nccl_unique_id: need a buffer of COLOC_NCCL_ID_BYTES bytes");
    auto const& a = api();
    if (!a.ok)
        return coloc_cuda::fail(COLOC_ERR_NCCL, a.why);
    ncclUniqueId id;
    ncclResult_t r = a.get_unique_id(&id);
    if (r != ncclSuccess)
        return nccl_fail(r, "ncclGetUniqueId");
    std::memcpy(id_out, &id, sizeof id);
    return COLOC_OK;
}

int coloc_cuda_nccl_init_rank(int dev, int nranks, const void* id, int rank, void** comm_out)
{
    if (!id || !comm_out || nranks <= 0 || rank < 0 || rank >= nranks)
        return coloc_cuda::fail(COLOC_ERR_INVALID_ARGUMENT, "nccl_init_rank: bad arguments");
    *comm_out = nullptr;
    auto const& a = api();
    if (!a.ok)
        return coloc_cuda::fail(COLOC_ERR_NCCL, a.why);
    COLOC_TRY(coloc_cuda::use_device(dev));
    ncclUniqueId uid;
    std::memcpy(&uid, id, sizeof uid);
    ncclComm_t c = nullptr;
    ncclResult_t r = a.comm_init_rank(&c, nranks, uid, rank);
    if (r != ncclSuccess)
        return nccl_fail(r, "ncclCommInitRank");
    *comm_out = c;
    return COLOC_OK;
}

int coloc_cuda_nccl_allreduce_f64(void* comm, int dev, void* stream, const double* send,
    double* recv, size_t count, int op)
{
    if (!comm || (!send && count) || (!recv && count))
        return coloc_cuda::fail(COLOC_ERR_INVALID_ARGUMENT, "nccl_allreduce_f64: bad arguments");
    ncclRedOp_t nop;
    switch (op)
    {
    case COLOC_REDUCE_SUM: nop = ncclSum; break;
    case COLOC_REDUCE_MAX: nop = ncclMax; break;
    case COLOC_REDUCE_MIN: nop = ncclMin; break;
    default: return coloc_cuda::fail(COLOC_ERR_INVALID_ARGUMENT, "nccl_allreduce_f64: unknown op");
    }
    auto const& a = api();
    if (!a.ok)
        return coloc_cuda::fail(COLOC_ERR_NCCL, a.why);
    COLOC_TRY(coloc_cuda::use_device(dev));
    ncclResult_t r = a.all_reduce(send, recv, count, ncclFloat64, nop, static_cast<ncclComm_t>(comm),
        static_cast<cudaStream_t>(stream));
    if (r != ncclSuccess)
        return nccl_fail(r, "ncclAllReduce");
    return COLOC_OK;
}

int coloc_cuda_nccl_destroy(int ndev, void* const* comms)
{
    if (ndev <= 0 || !comms)
        return COLOC_OK;
    auto const& a = api();
    if (!a.ok)
        return coloc_cuda::fail(COLOC_ERR_NCCL, a.why);
    for (int i = 0; i < ndev; ++i)
        if (comms[i])
            a.comm_destroy(static_cast<ncclComm_t>(comms[i]));
    return COLOC_OK;
}

}    // extern "C"
