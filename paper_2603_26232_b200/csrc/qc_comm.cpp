// Multi-GPU exchange of the QAOA stage: subgraphs are sharded in contiguous
// blocks across GPUs (qc_shard_range) and solved independently; the only collective is
// one all-gather of the fixed-size solve records, over NCCL (NVLink / NVSwitch on one
// box), after which the merge runs on the gathered records (qc_merge_records). This is
// what replaces pipeline.hpp:271-280 (one std::thread per subgraph per round) and the
// hand-over of the SolveResults to the merge at pipeline.hpp:300-305 for a C++ caller.
//
// NCCL is loaded at first use (dlopen "libnccl.so.2": the process's already-loaded copy,
// e.g. torch's, or the system one), so libqcgpu.so itself has no link-time NCCL
// dependency and the single-GPU paths never touch it.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <chrono>
#include <memory>
#include <cstring>
#include <mutex>
#include <string>
#include <thread>
#include <vector>

#include "qc_engine.hpp"

using namespace qcg;

namespace {

template <typename F>
int guarded(F&& f) {
    try {
        f();
        return QC_OK;
    } catch (const qcg::Error& e) {
        qcg::set_error(e.what());
        return e.code;
    } catch (const std::bad_alloc&) {
        qcg::set_error("host out of memory");
        return QC_ERR_RESOURCE;
    } catch (const std::exception& e) {
        qcg::set_error(e.what());
        return QC_ERR_INTERNAL;
    }
}

struct Nccl {
    ncclResult_t (*get_unique_id)(ncclUniqueId*) = nullptr;
    ncclResult_t (*comm_init_rank)(ncclComm_t*, int, ncclUniqueId, int) = nullptr;
    ncclResult_t (*comm_init_all)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*comm_destroy)(ncclComm_t) = nullptr;
    ncclResult_t (*all_gather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t, cudaStream_t) = nullptr;
    ncclResult_t (*group_start)() = nullptr;
    ncclResult_t (*group_end)() = nullptr;
    const char* (*error_string)(ncclResult_t) = nullptr;
};

const Nccl& nccl() {
    static Nccl n;
    static std::once_flag once;
    static std::string err;
    std::call_once(once, [] {
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) {
            err = std::string("NCCL not loadable: ") + dlerror();
            return;
        }
        auto sym = [&](const char* name) {
            void* p = dlsym(h, name);
            if (!p) err = std::string("NCCL symbol missing: ") + name;
            return p;
        };
        n.get_unique_id = reinterpret_cast<decltype(n.get_unique_id)>(sym("ncclGetUniqueId"));
        n.comm_init_rank = reinterpret_cast<decltype(n.comm_init_rank)>(sym("ncclCommInitRank"));
        n.comm_init_all = reinterpret_cast<decltype(n.comm_init_all)>(sym("ncclCommInitAll"));
        n.comm_destroy = reinterpret_cast<decltype(n.comm_destroy)>(sym("ncclCommDestroy"));
        n.all_gather = reinterpret_cast<decltype(n.all_gather)>(sym("ncclAllGather"));
        n.group_start = reinterpret_cast<decltype(n.group_start)>(sym("ncclGroupStart"));
        n.group_end = reinterpret_cast<decltype(n.group_end)>(sym("ncclGroupEnd"));
        n.error_string = reinterpret_cast<decltype(n.error_string)>(sym("ncclGetErrorString"));
    });
    if (!err.empty()) resource_error(err);
    return n;
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r == ncclSuccess) return;
    const char* s = nccl().error_string ? nccl().error_string(r) : "?";
    internal_error(std::string(what) + ": " + s);
}

}  // namespace

// One rank of a record-gather communicator: the NCCL communicator on the engine's device,
// ordered on the engine's stream, plus reusable device buffers for the padded records.
struct qc_comm {
    qc_engine* e = nullptr;
    ncclComm_t comm = nullptr;
    int nranks = 1, rank = 0;
    DevBuf send, recv;
    HostBuf hrecv;
};

extern "C" {

int qc_comm_id(void* id) {
    return guarded([&] {
        if (!id) config_error("null argument");
        ncclUniqueId u;
        nccl_check(nccl().get_unique_id(&u), "ncclGetUniqueId");
        std::memcpy(id, &u, sizeof(u));
    });
}

int qc_comm_create(qc_engine* e, int nranks, int rank, const void* id, qc_comm** out) {
    return guarded([&] {
        if (!e || !id || !out) config_error("null argument");
        if (nranks < 1 || rank < 0 || rank >= nranks) config_error("invalid rank/nranks");
        QC_CUDA(cudaSetDevice(e->device));
        auto c = std::make_unique<qc_comm>();
        c->e = e;
        c->nranks = nranks;
        c->rank = rank;
        ncclUniqueId u;
        std::memcpy(&u, id, sizeof(u));
        nccl_check(nccl().comm_init_rank(&c->comm, nranks, u, rank), "ncclCommInitRank");
        *out = c.release();
    });
}

int qc_comm_create_all(qc_engine* const* engines, int n, qc_comm** out) {
    return guarded([&] {
        if (!engines || !out || n < 1) config_error("null argument");
        std::vector<int> devs(static_cast<size_t>(n));
        for (int i = 0; i < n; ++i) {
            if (!engines[i]) config_error("null engine");
            devs[static_cast<size_t>(i)] = engines[i]->device;
            for (int j = 0; j < i; ++j)
                if (devs[static_cast<size_t>(j)] == devs[static_cast<size_t>(i)])
                    config_error("qc_comm_create_all needs one engine per distinct device");
        }
        std::vector<ncclComm_t> comms(static_cast<size_t>(n));
        nccl_check(nccl().comm_init_all(comms.data(), n, devs.data()), "ncclCommInitAll");
        for (int i = 0; i < n; ++i) {
            auto c = new qc_comm();
            c->e = engines[i];
            c->comm = comms[static_cast<size_t>(i)];
            c->nranks = n;
            c->rank = i;
            out[i] = c;
        }
    });
}

void qc_comm_destroy(qc_comm* c) {
    if (!c) return;
    cudaSetDevice(c->e->device);
    cudaStreamSynchronize(c->e->stream);
    if (c->comm) nccl().comm_destroy(c->comm);
    delete c;
}

int qc_comm_rank(const qc_comm* c, int32_t* rank, int32_t* nranks) {
    return guarded([&] {
        if (!c) config_error("null communicator");
        if (rank) *rank = c->rank;
        if (nranks) *nranks = c->nranks;
    });
}

}  // extern "C"

namespace {

// Stage this rank's records (padded to the largest shard) and enqueue the all-gather
// on the engine stream; collect() copies the gathered records back in subgraph order.
struct Gather {
    qc_comm* c;
    int M;
    int64_t rb;
    int32_t maxcount = 0;
    void enqueue(const void* local, int32_t count) {
        qc_engine* e = c->e;
        QC_CUDA(cudaSetDevice(e->device));
        maxcount = (M + c->nranks - 1) / c->nranks;  // qc_shard_range: ceil(M / nranks)
        if (count > maxcount) config_error("shard holds more records than its range");
        const size_t chunk = static_cast<size_t>(maxcount) * static_cast<size_t>(rb);
        void* s = c->send.get(std::max<size_t>(chunk, 1));
        void* r = c->recv.get(std::max<size_t>(chunk * static_cast<size_t>(c->nranks), 1));
        QC_CUDA(cudaMemsetAsync(s, 0, chunk, e->stream));
        if (count > 0)
            e->h2d_copy(s, local, static_cast<size_t>(count) * static_cast<size_t>(rb), e->stream);
        nccl_check(nccl().all_gather(s, r, chunk, ncclUint8, c->comm, e->stream), "ncclAllGather");
    }
    void collect(void* all) {
        qc_engine* e = c->e;
        QC_CUDA(cudaSetDevice(e->device));
        const size_t chunk = static_cast<size_t>(maxcount) * static_cast<size_t>(rb);
        char* h = static_cast<char*>(c->hrecv.get(std::max<size_t>(chunk * static_cast<size_t>(c->nranks), 1)));
        e->d2h_copy(h, c->recv.p, chunk * static_cast<size_t>(c->nranks), e->stream);
        QC_CUDA(cudaStreamSynchronize(e->stream));
        for (int r = 0; r < c->nranks; ++r) {
            int32_t b = 0, en = 0;
            if (qc_shard_range(M, r, c->nranks, &b, &en) != QC_OK) internal_error("shard range");
            std::memcpy(static_cast<char*>(all) + static_cast<int64_t>(b) * rb, h + static_cast<size_t>(r) * chunk,
                        static_cast<size_t>(en - b) * static_cast<size_t>(rb));
        }
    }
};

}  // namespace

extern "C" {

int qc_gather_topk(qc_comm* c, const void* local, int32_t count, int32_t M, int64_t record_bytes,
                   void* all) {
    return guarded([&] {
        if (!c || !all || (count > 0 && !local)) config_error("null argument");
        if (M < 0 || record_bytes < 1) config_error("invalid record geometry");
        int32_t b = 0, en = 0;
        if (qc_shard_range(M, c->rank, c->nranks, &b, &en) != QC_OK) config_error("invalid shard request");
        if (count != en - b)
            config_error("rank " + std::to_string(c->rank) + " holds " + std::to_string(count) +
                         " records, its shard [" + std::to_string(b) + ", " + std::to_string(en) + ") has " +
                         std::to_string(en - b));
        NvtxRange nv("qcgpu.gather_topk");
        Gather gth{c, M, record_bytes};
        gth.enqueue(local, count);
        gth.collect(all);
    });
}

// One process driving n GPUs (one engine each): shard -> solve (one host thread per
// engine) -> NCCL all-gather of the records -> merge on engines[0].
int qc_run_pipeline_multi(qc_engine* const* engines, qc_comm* const* comms, int n, const qc_graph* g,
                          const qc_run_config* cfg, qc_run_report* report, char* assignment) {
    return guarded([&] {
        if (!engines || !cfg || n < 1) config_error("null argument");
        int64_t rb = 0;
        int32_t M = 0;
        {
            const int rc = qc_run_record_bytes(g, cfg, &rb, &M);
            if (rc != QC_OK) throw Error(rc, qc_last_error());
        }
        for (int i = 0; i < n; ++i)
            if (!engines[i]) config_error("null engine");
        if (comms)
            for (int i = 0; i < n; ++i)
                if (!comms[i] || comms[i]->e != engines[i] || comms[i]->rank != i || comms[i]->nranks != n)
                    config_error("comms[i] must be rank i of an n-rank communicator on engines[i]");
        std::vector<char> all(static_cast<size_t>(std::max<int64_t>(rb * M, 1)));
        std::vector<std::vector<char>> local(static_cast<size_t>(n));
        std::vector<int> rc(static_cast<size_t>(n), QC_OK);
        std::vector<std::string> msg(static_cast<size_t>(n));
        std::vector<int32_t> begin(static_cast<size_t>(n)), end(static_cast<size_t>(n));
        const auto t0 = std::chrono::steady_clock::now();
        auto work = [&](int i) {
            const size_t k = static_cast<size_t>(i);
            qc_run_config c = *cfg;
            c.shard_index = i;
            c.shard_count = n;
            rc[k] = qc_shard_range(M, i, n, &begin[k], &end[k]);
            if (rc[k] == QC_OK) {
                local[k].assign(static_cast<size_t>(std::max<int64_t>(rb * (end[k] - begin[k]), 1)), 0);
                rc[k] = qc_shard_solve(engines[i], g, &c, begin[k], end[k], local[k].data(),
                                       static_cast<int64_t>(local[k].size()), nullptr);
            }
            if (rc[k] != QC_OK) msg[k] = qc_last_error();
        };
        // one host thread per DISTINCT engine (an engine is driven by one thread at a time):
        // shards that share an engine object run back to back on that engine's thread
        std::vector<std::vector<int>> by_engine;
        for (int i = 0; i < n; ++i) {
            bool placed = false;
            for (auto& grp : by_engine)
                if (engines[grp[0]] == engines[i]) {
                    grp.push_back(i);
                    placed = true;
                    break;
                }
            if (!placed) by_engine.push_back({i});
        }
        if (comms && by_engine.size() != static_cast<size_t>(n))
            config_error("an NCCL communicator needs one engine per rank");
        auto run_group = [&](size_t gi) {
            for (int i : by_engine[gi]) work(i);
        };
        std::vector<std::thread> ts;
        for (size_t gi = 1; gi < by_engine.size(); ++gi) ts.emplace_back(run_group, gi);
        run_group(0);
        for (auto& t : ts) t.join();
        for (int i = 0; i < n; ++i)
            if (rc[static_cast<size_t>(i)] != QC_OK) throw Error(rc[static_cast<size_t>(i)], msg[static_cast<size_t>(i)]);
        const double qaoa_s = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
        if (comms) {
            // every rank's all-gather must be in flight together (one NCCL group)
            std::vector<Gather> gs;
            for (int i = 0; i < n; ++i) gs.push_back(Gather{comms[i], M, rb});
            nccl_check(nccl().group_start(), "ncclGroupStart");
            try {
                for (int i = 0; i < n; ++i)
                    gs[static_cast<size_t>(i)].enqueue(local[static_cast<size_t>(i)].data(),
                                                       end[static_cast<size_t>(i)] - begin[static_cast<size_t>(i)]);
            } catch (...) {
                nccl().group_end();
                throw;
            }
            nccl_check(nccl().group_end(), "ncclGroupEnd");
            gs[0].collect(all.data());  // every rank now holds all M records; rank 0 merges
            for (int i = 1; i < n; ++i) QC_CUDA(cudaStreamSynchronize(engines[i]->stream));
        } else {
            // engines sharing a device cannot form an NCCL communicator: the records are
            // already in host memory, so they are concatenated in subgraph order
            for (int i = 0; i < n; ++i)
                std::memcpy(all.data() + static_cast<int64_t>(begin[static_cast<size_t>(i)]) * rb,
                            local[static_cast<size_t>(i)].data(),
                            static_cast<size_t>(end[static_cast<size_t>(i)] - begin[static_cast<size_t>(i)]) * static_cast<size_t>(rb));
        }
        qc_run_config c0 = *cfg;
        c0.shard_index = 0;
        c0.shard_count = 1;
        qc_run_report r{};
        const int mrc = qc_merge_records(engines[0], g, &c0, all.data(), rb * M, M, &r, assignment);
        if (mrc != QC_OK) throw Error(mrc, qc_last_error());
        r.qaoa_s = qaoa_s;
        r.total_s = r.partition_s + r.qaoa_s + r.merge_s;
        if (report) *report = r;
    });
}

}  // extern "C"
