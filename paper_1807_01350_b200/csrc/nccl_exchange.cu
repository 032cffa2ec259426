// Library-owned collectives of a sharded stream: the
// reference's parallel_replicas join (proj/src/streaming.cpp:45-69) across
// GPUs, as NCCL collectives on the stream's own CUDA stream.
//
//   replica sharding   begin -> ncclAllGather(models) -> merge
//                            -> ncclAllGather(temporal-stack rows) -> finish
//   temporal sharding  begin_temporal -> ncclReduceScatter(partial summaries)
//                            -> begin_reduced -> the same two all-gathers
//
// NCCL is resolved at run time (dlopen of libnccl.so.2): a process that
// already loaded NCCL (e.g. PyTorch's) shares that library, otherwise the
// system one is loaded.  A communicator is created from a unique id the
// caller distributes (octen_nccl_get_unique_id), or an existing ncclComm_t
// is borrowed.
#include <cuda_runtime.h>
#include <dlfcn.h>
#include <nccl.h>

#include <cstring>
#include <mutex>
#include <string>

#include "errors.hpp"
#include "stream.hpp"

namespace octen {

namespace {

struct NcclApi {
    ncclResult_t (*GetUniqueId)(ncclUniqueId*) = nullptr;
    ncclResult_t (*CommInitRank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*CommDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*AllGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*ReduceScatter)(const void*, void*, size_t, ncclDataType_t, ncclRedOp_t, ncclComm_t,
                                  cudaStream_t) = nullptr;
    const char* (*GetErrorString)(ncclResult_t) = nullptr;
    ncclResult_t (*GetVersion)(int*) = nullptr;
    bool ok = false;
    std::string why;
};

NcclApi& nccl() {
    static NcclApi api;
    static std::once_flag once;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_NOLOAD);  // already in the process (e.g. PyTorch's)
        if (!h) h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            const char* e = dlerror();
            api.why = std::string("octen: NCCL is not available (") + (e ? e : "libnccl.so.2 not found") + ")";
            return;
        }
        auto sym = [&](const char* n) { return dlsym(h, n); };
        api.GetUniqueId = reinterpret_cast<decltype(api.GetUniqueId)>(sym("ncclGetUniqueId"));
        api.CommInitRank = reinterpret_cast<decltype(api.CommInitRank)>(sym("ncclCommInitRank"));
        api.CommDestroy = reinterpret_cast<decltype(api.CommDestroy)>(sym("ncclCommDestroy"));
        api.AllGather = reinterpret_cast<decltype(api.AllGather)>(sym("ncclAllGather"));
        api.ReduceScatter = reinterpret_cast<decltype(api.ReduceScatter)>(sym("ncclReduceScatter"));
        api.GetErrorString = reinterpret_cast<decltype(api.GetErrorString)>(sym("ncclGetErrorString"));
        api.GetVersion = reinterpret_cast<decltype(api.GetVersion)>(sym("ncclGetVersion"));
        api.ok = api.GetUniqueId && api.CommInitRank && api.CommDestroy && api.AllGather && api.ReduceScatter &&
                 api.GetErrorString;
        if (!api.ok) api.why = "octen: libnccl.so.2 lacks the collectives this library calls";
    });
    if (!api.ok) throw CudaError(api.why);
    return api;
}

void check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess) throw CudaError(std::string("octen: ") + what + ": " + nccl().GetErrorString(r));
}

}  // namespace

NcclExchange::~NcclExchange() {
    if (comm && owned) nccl().CommDestroy(static_cast<ncclComm_t>(comm));
}

void nccl_unique_id(unsigned char* out128) {
    static_assert(sizeof(ncclUniqueId) == 128, "ncclUniqueId is 128 bytes");
    ncclUniqueId id;
    check(nccl().GetUniqueId(&id), "ncclGetUniqueId");
    std::memcpy(out128, &id, 128);
}

void Stream::attach_nccl(const unsigned char* uid128, void* borrowed_comm) {
    if (shard_world < 1) throw ConfigError("octen: bad shard world");
    auto x = std::make_unique<NcclExchange>();
    if (borrowed_comm) {
        x->comm = borrowed_comm;
        x->owned = false;
    } else {
        ncclUniqueId id;
        std::memcpy(&id, uid128, 128);
        ncclComm_t c = nullptr;
        OCTEN_CUDA(cudaSetDevice(cfg.device));
        check(nccl().CommInitRank(&c, shard_world, id, shard_rank), "ncclCommInitRank");
        x->comm = c;
        x->owned = true;
    }
    nccl_x = std::move(x);
}

void Stream::exchange_allgather(const double* send, double* recv, size_t count) {
    check(nccl().AllGather(send, recv, count, ncclFloat64, static_cast<ncclComm_t>(nccl_x->comm), st),
          "ncclAllGather");
}

void Stream::ingest_sharded(const void* data, int dtype, int location, int order, const std::int64_t* dims) {
    if (!nccl_x) throw ConfigError("octen: the stream has no NCCL communicator (octen_stream_create_nccl)");
    const size_t mc = models_count(), rc = rows_count();
    xmodels.reserve(mc);
    xmodels2.reserve(mc * shard_world);
    xrows.reserve(rc);
    DevBuf<double>& rows_all = rows_all_buf;
    rows_all.reserve(rc * shard_world);
    begin(cur, data, dtype, location, order, dims, xmodels.p, false);
    exchange_allgather(xmodels.p, xmodels2.p, mc);  // on st: the merge reads after it
    merge_phase(cur, xmodels2.p, xrows.p);
    exchange_allgather(xrows.p, rows_all.p, rc);
    finish(cur, rows_all.p);
}

void Stream::ingest_temporal_nccl(const void* data, int dtype, int location, int order,
                                  const std::int64_t* dims_local, std::int64_t k_off, std::int64_t t_total) {
    if (!nccl_x) throw ConfigError("octen: the stream has no NCCL communicator (octen_stream_create_nccl)");
    const size_t blk = partial_block_count();
    DevBuf<double>& part = part_buf;
    DevBuf<double>& owned = owned_buf;
    part.reserve(blk * shard_world);
    owned.reserve(blk);
    begin_temporal(data, dtype, location, order, dims_local, k_off, t_total, part.p);
    // sum over ranks of their partials of this rank's replicas (the status
    // slot sums the ranks' non-finite flags)
    check(nccl().ReduceScatter(part.p, owned.p, blk, ncclFloat64, ncclSum, static_cast<ncclComm_t>(nccl_x->comm), st),
          "ncclReduceScatter");
    const size_t mc = models_count(), rc = rows_count();
    xmodels.reserve(mc);
    xmodels2.reserve(mc * shard_world);
    xrows.reserve(rc);
    rows_all_buf.reserve(rc * shard_world);
    begin_reduced(owned.p, xmodels.p);
    exchange_allgather(xmodels.p, xmodels2.p, mc);
    merge_phase(cur, xmodels2.p, xrows.p);
    exchange_allgather(xrows.p, rows_all_buf.p, rc);
    finish(cur, rows_all_buf.p);
}

}  // namespace octen
