// sharded.cpp -- one logical ExperienceBuffer / ParetoFrontier over the GPUs of
// one process, inside the C ABI (sharded.py is the mirror for
// one process per GPU over torch.distributed).  The C++ drop-in can therefore
// spread a buffer over the node's GPUs without Python.
//
// Layout: shard r (device r of the communicator) holds the contiguous global
// records [lo_r, lo_r + n_r); appends fill the shards in order, quota records
// each (capacity / shards), so global indices -- the reference's tie-break --
// are the insertion order, as in one buffer.  Exactness rests on the same
// three exchanges as sharded.py:
//   statistics  the shards' running sums combined in shard order;
//   sigma       the buffer's 512-row subsample (experience.cpp:82-91) gathered
//               from the owning shards, the median on device 0, under the
//               reference's cache state machine (:116-121, refresh every 50
//               stored records);
//   candidates  every shard selects its top-m with the buffer's statistics
//               (concurrently, one host thread per device); the per-shard
//               packs are all-gathered device to device (NCCL over NVLink when
//               the shards sit on distinct GPUs, ncclCommInitAll; peer copies
//               otherwise) and merged on device 0 (merge_packed: score desc,
//               round asc, global index asc, then curriculum order).
// lambda != 0: every greedy step's arg-max is taken across the shards
// (greedy_begin / greedy_next: each shard's best with its row; the winner by
// gain desc, round asc, index asc; every shard adds its similarity).
// Pareto: each shard reduces its slice of a batch to a local frontier on its
// device (K6), the local frontiers are inserted into the buffer's frontier --
// the frontier of a union is the frontier of the union of frontiers.
#include <dlfcn.h>
#include <nccl.h>

#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>
#include <exception>
#include <thread>
#include <vector>

#include "internal.hpp"

namespace sair {
namespace {

// NCCL through dlopen: libsair carries no link-time NCCL dependency (the
// library loaded by the host process -- torch's, or the system's -- is used)
struct NcclApi {
    bool ok = false;
    ncclResult_t (*commInitAll)(ncclComm_t*, int, const int*) = nullptr;
    ncclResult_t (*commDestroy)(ncclComm_t) = nullptr;
    ncclResult_t (*allGather)(const void*, void*, size_t, ncclDataType_t, ncclComm_t,
                              cudaStream_t) = nullptr;
    ncclResult_t (*groupStart)() = nullptr;
    ncclResult_t (*groupEnd)() = nullptr;
    const char* (*errorString)(ncclResult_t) = nullptr;
};

NcclApi& nccl_api() {
    static NcclApi api = [] {
        NcclApi a;
        void* h = dlopen("libnccl.so.2", RTLD_NOW | RTLD_GLOBAL);
        if (!h) h = dlopen("libnccl.so", RTLD_NOW | RTLD_GLOBAL);
        if (!h) return a;
        a.commInitAll = reinterpret_cast<decltype(a.commInitAll)>(dlsym(h, "ncclCommInitAll"));
        a.commDestroy = reinterpret_cast<decltype(a.commDestroy)>(dlsym(h, "ncclCommDestroy"));
        a.allGather = reinterpret_cast<decltype(a.allGather)>(dlsym(h, "ncclAllGather"));
        a.groupStart = reinterpret_cast<decltype(a.groupStart)>(dlsym(h, "ncclGroupStart"));
        a.groupEnd = reinterpret_cast<decltype(a.groupEnd)>(dlsym(h, "ncclGroupEnd"));
        a.errorString = reinterpret_cast<decltype(a.errorString)>(dlsym(h, "ncclGetErrorString"));
        a.ok = a.commInitAll && a.commDestroy && a.allGather && a.groupStart && a.groupEnd &&
               a.errorString;
        return a;
    }();
    return api;
}

// fn(r) for every shard r on its own host thread (each drives its device);
// the first exception is rethrown after all have joined
template <class F>
void for_shards(size_t S, F&& fn) {
    std::vector<std::exception_ptr> err(S);
    std::vector<std::thread> th;
    for (size_t r = 0; r < S; ++r)
        th.emplace_back([&, r] {
            try {
                fn(r);
            } catch (...) {
                err[r] = std::current_exception();
            }
        });
    for (auto& t : th) t.join();
    for (auto& e : err)
        if (e) std::rethrow_exception(e);
}

void nccl_check(ncclResult_t r, const char* what) {
    if (r != ncclSuccess)
        throw Error(SAIR_ENCCL, std::string(what) + ": " + nccl_api().errorString(r));
}

}  // namespace
}  // namespace sair

namespace sair {

void comm_create(const int* devices, int n, sair_comm_s* c) {
    int ndev = 0;
    if (cudaGetDeviceCount(&ndev) != cudaSuccess || ndev == 0)
        throw Error(SAIR_ECUDA, "no CUDA device (libsair has no CPU fallback)");
    if (n < 1) throw Error(SAIR_EINVAL, "comm: at least one device");
    for (int i = 0; i < n; ++i)
        if (devices[i] < 0 || devices[i] >= ndev) throw Error(SAIR_EINVAL, "comm: bad device id");
    c->dev.assign(devices, devices + n);
    for (int i = 0; i < n; ++i) {
        DeviceGuard g(c->dev[i]);
        cudaStream_t s;
        SAIR_CUDA(cudaStreamCreateWithFlags(&s, cudaStreamNonBlocking));
        c->st.push_back(s);
    }
    std::vector<int> u(c->dev);
    std::sort(u.begin(), u.end());
    const bool distinct = std::unique(u.begin(), u.end()) == u.end();
    // (SAIR_COMM_NCCL=1: NCCL even for one device -- exercises the transport
    // on a single GPU)
    const char* fe = std::getenv("SAIR_COMM_NCCL");
    if (distinct && (n > 1 || (fe && std::atoi(fe) == 1))) {
        // one communicator over the process's GPUs (NVLink / NVSwitch)
        if (!nccl_api().ok) throw Error(SAIR_ENCCL, "comm: libnccl.so.2 not loadable");
        std::vector<ncclComm_t> nc(n);
        nccl_check(nccl_api().commInitAll(nc.data(), n, c->dev.data()), "ncclCommInitAll");
        c->nc.assign(nc.begin(), nc.end());
    }
}

void comm_free(sair_comm_s* c) {
    for (auto x : c->nc) nccl_api().commDestroy(static_cast<ncclComm_t>(x));
    for (size_t i = 0; i < c->st.size(); ++i) {
        DeviceGuard g(c->dev[i]);
        cudaStreamDestroy(c->st[i]);
    }
}

// recv[r] (device r) <- the concatenation of every send[j] (bytes each, shard order)
void comm_allgather(sair_comm_s* c, const std::vector<const void*>& send,
                    const std::vector<void*>& recv, size_t bytes) {
    const int n = (int)c->dev.size();
    if (!c->nc.empty()) {
        auto& api = nccl_api();
        nccl_check(api.groupStart(), "ncclGroupStart");
        for (int r = 0; r < n; ++r) {
            DeviceGuard g(c->dev[r]);
            nccl_check(api.allGather(send[r], recv[r], bytes, ncclChar, static_cast<ncclComm_t>(c->nc[r]), c->st[r]),
                       "ncclAllGather");
        }
        nccl_check(api.groupEnd(), "ncclGroupEnd");
    } else {  // one device (or shards sharing devices): unified-address copies
        for (int r = 0; r < n; ++r) {
            DeviceGuard g(c->dev[r]);
            for (int j = 0; j < n; ++j)
                SAIR_CUDA(cudaMemcpyAsync(static_cast<char*>(recv[r]) + (size_t)j * bytes, send[j],
                                          bytes, cudaMemcpyDefault, c->st[r]));
        }
    }
    for (int r = 0; r < n; ++r) {
        DeviceGuard g(c->dev[r]);
        SAIR_CUDA(cudaStreamSynchronize(c->st[r]));
    }
}

void sharded_init(sair_sharded_s* h, sair_comm_s* c, double r_min, size_t capacity) {
    h->comm = c;
    h->r_min = r_min;
    const size_t S = c->dev.size();
    h->quota = std::max<size_t>(1, (std::max<size_t>(capacity, 1) + S - 1) / S);
    h->b_pack.resize(S);
    for (size_t r = 0; r < S; ++r) {
        auto* s = new sair_store_s();
        try {
            store_init(s, r_min, c->dev[r], std::min(h->quota, (size_t)1 << 20));
        } catch (...) {
            delete s;
            throw;
        }
        h->sh.push_back(s);
        h->lo.push_back(0);
    }
}

void sharded_free(sair_sharded_s* h) {
    for (auto* s : h->sh) {
        store_free(s);
        delete s;
    }
    h->sh.clear();
}

// store() of count rows, in order: the gate, then the shards in order
// (experience.cpp:44-62: rejected rows only count; the first accepted row
// fixes the dimension)
size_t sharded_append(sair_sharded_s* h, const double* ctx, size_t count, int dim,
                      const double* reward, const int32_t* round, uint8_t* accepted) {
    std::vector<size_t> acc;
    acc.reserve(count);
    for (size_t i = 0; i < count; ++i) {
        const bool ok = reward[i] > h->r_min;
        if (accepted) accepted[i] = ok ? 1 : 0;
        if (!ok) {
            ++h->rejected;
            continue;
        }
        if (h->n + acc.size() == 0) {
            h->d = dim;
            h->gst.sum.assign(dim, 0.0);
            h->gst.sum_sq.assign(dim, 0.0);
            h->gst.xabs.assign(dim, 0.0);
        } else if (dim != h->d) {
            throw Error(SAIR_EINVAL, "experience store: context dimension changed");
        }
        acc.push_back(i);
    }
    for (size_t i : acc) {  // the same additions, the same order as one buffer
        const double* x = ctx + i * (size_t)dim;
        for (int j = 0; j < dim; ++j) {
            h->gst.sum[j] += x[j];
            h->gst.sum_sq[j] += x[j] * x[j];
            h->gst.xabs[j] = std::max(h->gst.xabs[j], std::fabs(x[j]));
        }
        h->gst.total += reward[i];
        h->gst.rabs = std::max(h->gst.rabs, std::fabs(reward[i]));
    }
    std::vector<double> x, r;
    std::vector<int32_t> rd;
    size_t k = 0;
    const size_t S = h->sh.size();
    while (k < acc.size()) {
        // the first shard with room (the last one takes any overflow)
        size_t s = 0;
        while (s + 1 < S && h->sh[s]->n >= h->quota) ++s;
        if (h->sh[s]->n == 0) {
            h->lo[s] = h->n;
            h->sh[s]->gbase = (int64_t)h->n;
        }
        const size_t room = s + 1 < S ? h->quota - h->sh[s]->n : acc.size() - k;
        const size_t take = std::min(room, acc.size() - k);
        x.resize(take * dim);
        r.resize(take);
        rd.resize(take);
        for (size_t j = 0; j < take; ++j) {
            const size_t i = acc[k + j];
            std::memcpy(x.data() + j * dim, ctx + i * (size_t)dim, (size_t)dim * 8);
            r[j] = reward[i];
            rd[j] = round ? round[i] : (int32_t)(h->n + j);
        }
        store_append(h->sh[s], x.data(), take, dim, r.data(), rd.data(), nullptr);
        h->n += take;
        h->stale += take;  // ++sigma_stale_count_ per stored record
        k += take;
    }
    return acc.size();
}

void sharded_append_synthetic(sair_sharded_s* h, uint64_t seed, size_t count, int dim,
                              int clustered) {
    if (h->n && dim != h->d) throw Error(SAIR_EINVAL, "experience store: context dimension changed");
    const size_t S = h->sh.size();
    size_t k = 0;
    while (k < count) {
        size_t s = 0;
        while (s + 1 < S && h->sh[s]->n >= h->quota) ++s;
        if (h->sh[s]->n == 0) {
            h->lo[s] = h->n;
            h->sh[s]->gbase = (int64_t)h->n;
        }
        const size_t room = s + 1 < S ? h->quota - h->sh[s]->n : count - k;
        const size_t take = std::min(room, count - k);
        // the generator is counter-based on the global index: record gbase + i;
        // its partial sums are exact, so adding the shard's increment is too
        const StoreStats before = h->sh[s]->stats;
        store_append_synthetic(h->sh[s], seed, take, dim, clustered);
        const StoreStats& after = h->sh[s]->stats;
        if (h->gst.sum.empty()) {
            h->gst.sum.assign(dim, 0.0);
            h->gst.sum_sq.assign(dim, 0.0);
            h->gst.xabs.assign(dim, 0.0);
        }
        for (int k2 = 0; k2 < dim; ++k2) {
            h->gst.sum[k2] += after.sum[k2] - (before.sum.empty() ? 0.0 : before.sum[k2]);
            h->gst.sum_sq[k2] += after.sum_sq[k2] - (before.sum_sq.empty() ? 0.0 : before.sum_sq[k2]);
            h->gst.xabs[k2] = std::max(h->gst.xabs[k2], after.xabs[k2]);
        }
        h->gst.total += after.total - before.total;
        h->gst.rabs = std::max(h->gst.rabs, after.rabs);
        h->n += take;
        h->stale += take;
        h->d = dim;
        k += take;
    }
}

// the buffer's statistics and sigma into every non-empty shard (global mode)
void sharded_sync(sair_sharded_s* h, double sigma_sim) {
    const int d = h->d;
    const StoreStats& g = h->gst;
    // sigma: experience.cpp:116-121 at the buffer level
    double sigma = 1.0;
    if (sigma_sim > 0.0) {
        sigma = sigma_sim;
    } else if (h->n >= 2) {
        if (h->cached_sigma == 0.0 || h->stale >= 50) {
            // moments from the combined sums (store_mean_sd on a global-mode shard)
            for (auto* s : h->sh)
                if (s->n) {
                    s->sharded = true;
                    s->n_global = h->n;
                    s->gst = g;
                    s->gsigma = 1.0;
                }
            std::vector<double> mean(d), sd(d);
            for (auto* s : h->sh)
                if (s->n) {
                    store_mean_sd(s, mean.data(), sd.data());
                    break;
                }
            const auto idx = sigma_sample(h->n);
            std::vector<double> rows(idx.size() * d);
            for (size_t j = 0; j < idx.size(); ++j) {
                size_t r = 0;
                while (r + 1 < h->sh.size() && h->sh[r + 1]->n && (size_t)idx[j] >= h->lo[r + 1]) ++r;
                sair_store_s* s = h->sh[r];
                DeviceGuard dg(s->device);
                SAIR_CUDA(cudaMemcpy(rows.data() + j * d, s->x64 + ((size_t)idx[j] - h->lo[r]) * d,
                                     (size_t)d * 8, cudaMemcpyDeviceToHost));
            }
            h->cached_sigma =
                idx.size() >= 2 ? sigma_rows(rows.data(), idx.size(), d, mean.data(), sd.data(),
                                             h->comm->dev[0])
                                : 1.0;
            h->stale = 0;
        }
        sigma = h->cached_sigma;
    }
    for (auto* s : h->sh)
        if (s->n) {
            s->sharded = true;
            s->n_global = h->n;
            s->gst = g;
            s->gsigma = sigma;
        }
    h->synced_n = h->n;
    h->synced_sigma = sigma;
}

void sharded_select(sair_sharded_s* h, const double* q, size_t nq, int dim,
                    const sair_select_config& cfg, int64_t* out_idx, double* out_sim,
                    double* out_score, size_t* out_count) {
    const size_t m = cfg.m;
    if (nq == 0) return;
    if (h->n == 0 || m == 0) {
        std::fill(out_count, out_count + nq, (size_t)0);
        return;
    }
    if (dim != h->d) throw Error(SAIR_EINVAL, "experience store: feature dimension mismatch");
    sharded_sync(h, cfg.sigma_sim);
    const size_t S = h->sh.size();
    if (cfg.lambda_div != 0.0) {
        // the distributed greedy: one arg-max across the shards per step
        const size_t want = std::min(m, h->n);
        const int d = h->d;
        const size_t W = 6 + d;
        std::vector<std::vector<double>> best(S, std::vector<double>(nq * W));
        for_shards(S, [&](size_t r) {
            if (h->sh[r]->n) greedy_begin(h->sh[r], q, nq, dim, cfg, best[r].data());
        });
        std::vector<std::vector<double>> picks(nq);
        std::vector<int64_t> gp(nq);
        std::vector<double> rows(nq * d);
        for (size_t step = 0; step < want; ++step) {
            for (size_t qq = 0; qq < nq; ++qq) {
                const double* w = nullptr;
                for (size_t r = 0; r < S; ++r) {
                    if (!h->sh[r]->n) continue;
                    const double* c = best[r].data() + qq * W;
                    if (c[2] < 0) continue;  // no untaken record on the shard
                    // gain desc, round asc, global index asc (experience.cpp:177-187)
                    if (!w || c[0] > w[0] || (c[0] == w[0] && (c[1] < w[1] ||
                                                              (c[1] == w[1] && c[2] < w[2]))))
                        w = c;
                }
                picks[qq].insert(picks[qq].end(), w, w + 6);
                gp[qq] = (int64_t)w[2];
                std::memcpy(rows.data() + qq * d, w + 6, (size_t)d * 8);
            }
            if (step + 1 == want) break;
            for_shards(S, [&](size_t r) {
                if (h->sh[r]->n) greedy_next(h->sh[r], gp.data(), rows.data(), best[r].data());
            });
        }
        // curriculum order (experience.cpp:197-204): reward asc, round asc, stable
        for (size_t qq = 0; qq < nq; ++qq) {
            std::vector<size_t> o(want);
            for (size_t x = 0; x < want; ++x) o[x] = x;
            const double* P = picks[qq].data();
            std::stable_sort(o.begin(), o.end(), [&](size_t a, size_t b) {
                if (P[a * 6 + 5] != P[b * 6 + 5]) return P[a * 6 + 5] < P[b * 6 + 5];
                return P[a * 6 + 1] < P[b * 6 + 1];
            });
            for (size_t x = 0; x < want; ++x) {
                out_idx[qq * m + x] = (int64_t)P[o[x] * 6 + 2];
                out_sim[qq * m + x] = P[o[x] * 6 + 3];
                out_score[qq * m + x] = P[o[x] * 6 + 4];
            }
            out_count[qq] = want;
        }
        return;
    }
    // lambda == 0: each shard's top-m (concurrently), packed as sharded.py
    // packs them -- [nq][5m + 1]: score | sim | reward | gidx | round | count
    const size_t PW = 5 * m + 1;
    std::vector<std::vector<double>> pack(S, std::vector<double>(nq * PW, 0.0));
    for_shards(S, [&](size_t r) {
            sair_store_s* s = h->sh[r];
            double* P = pack[r].data();
            if (!s->n) return;  // an empty shard contributes count 0
            std::vector<int64_t> idx(nq * m, -1);
            std::vector<double> sim(nq * m), sc(nq * m), rw(nq * m);
            std::vector<int32_t> rd(nq * m);
            std::vector<size_t> cnt(nq);
            store_select(s, q, nq, dim, cfg, idx.data(), sim.data(), sc.data(), cnt.data(),
                         nullptr, nullptr, rw.data(), rd.data());
            for (size_t qq = 0; qq < nq; ++qq) {
                double* row = P + qq * PW;
                for (size_t x = 0; x < m; ++x) {
                    row[x] = sc[qq * m + x];
                    row[m + x] = sim[qq * m + x];
                    row[2 * m + x] = rw[qq * m + x];
                    row[3 * m + x] = (double)idx[qq * m + x];
                    row[4 * m + x] = (double)rd[qq * m + x];
                }
                row[5 * m] = (double)cnt[qq];
            }
        });
    // device-resident packs, all-gathered to every device (NCCL), merged on device 0
    const size_t pb = nq * PW * 8;
    std::vector<const void*> send(S);
    std::vector<void*> recv(S);
    double* merged = nullptr;
    for (size_t r = 0; r < S; ++r) {
        DeviceGuard g(h->comm->dev[r]);
        char* b = static_cast<char*>(h->b_pack[r].get(pb * (S + 1) + nq * (3 * m + 1) * 8 + 512));
        SAIR_CUDA(cudaMemcpyAsync(b, pack[r].data(), pb, cudaMemcpyHostToDevice, h->comm->st[r]));
        send[r] = b;
        recv[r] = b + pb;
        if (r == 0) merged = reinterpret_cast<double*>(b + pb * (S + 1));
        SAIR_CUDA(cudaStreamSynchronize(h->comm->st[r]));
    }
    comm_allgather(h->comm, send, recv, pb);
    merge_packed(static_cast<const double*>(recv[0]), S, nq, m, h->comm->dev[0], h->comm->st[0], merged);
    std::vector<double> out(nq * (3 * m + 1));
    {
        DeviceGuard g(h->comm->dev[0]);
        SAIR_CUDA(cudaMemcpyAsync(out.data(), merged, out.size() * 8, cudaMemcpyDeviceToHost,
                                  h->comm->st[0]));
        SAIR_CUDA(cudaStreamSynchronize(h->comm->st[0]));
    }
    for (size_t qq = 0; qq < nq; ++qq) {
        const double* o = out.data() + qq * (3 * m + 1);
        const size_t c = (size_t)o[3 * m];
        out_count[qq] = c;
        for (size_t x = 0; x < c; ++x) {
            out_idx[qq * m + x] = (int64_t)o[x];
            out_sim[qq * m + x] = o[m + x];
            out_score[qq * m + x] = o[2 * m + x];
        }
    }
}

double sharded_effective_sigma(sair_sharded_s* h, double sigma_sim) {
    if (h->n == 0) return sigma_sim > 0.0 ? sigma_sim : 1.0;
    sharded_sync(h, sigma_sim);
    return h->synced_sigma;
}

// insert_normalized() of T tuples into f: each device reduces its slice to a
// local frontier (K6), the local frontiers go into f in shard order
size_t frontier_insert_batch_sharded(sair_comm_s* c, sair_frontier_s* f, const double* pts,
                                     size_t T) {
    const size_t S = c->dev.size();
    std::vector<std::vector<double>> loc(S);
    for_shards(S, [&](size_t r) {
            const size_t a = T * r / S, b = T * (r + 1) / S;
            if (a == b) return;
            sair_frontier_s lf;
            frontier_init(&lf, f->l_max, f->c_max, c->dev[r]);
            try {
                frontier_insert_batch(&lf, pts + 2 * a, b - a);
                loc[r].resize(2 * lf.F);
                for (size_t i = 0; i < lf.F; ++i) {
                    loc[r][2 * i] = lf.hl[i];
                    loc[r][2 * i + 1] = lf.hc[i];
                }
            } catch (...) {
                frontier_free(&lf);
                throw;
            }
            frontier_free(&lf);
        });
    std::vector<double> all;
    for (auto& v : loc) all.insert(all.end(), v.begin(), v.end());
    return frontier_insert_batch(f, all.data(), all.size() / 2);
}

}  // namespace sair
