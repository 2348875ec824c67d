// runtime.cpp -- trajectory executor and the device entry points of the C ABI.
//
// qt_run_trajectories processes `batch` trajectories at a time:
//   host  : plan every trajectory of the batch in parallel (planner.cpp),
//           concatenate the programs into pinned staging buffers;
//   device: upload, K6 materialize fused matrices, K1 tile passes step by step
//           (pass j of every trajectory in one launch; rho_Q + choose happen in
//           K1 epilogues, so there is no host round trip inside a batch),
//           K4 finalize observables, K3 sample bitstrings, download records.
// While the GPU runs batch i the host plans batch i+1 (two staging slots).
#include <cuda_runtime.h>
#include <nvtx3/nvToolsExt.h>

#include <algorithm>
#include <array>
#include <cstdio>
#include <cstdlib>
#include <chrono>
#include <cmath>
#include <cstring>
#include <memory>
#include <string>
#include <thread>
#include <vector>

#include "host.hpp"
#include "kernels.hpp"

namespace qt {
const Plan& plan_of(qt_plan p);
}

using namespace qt;

namespace {

#define QT_CK(expr)                                                                  \
    do {                                                                             \
        cudaError_t _e = (expr);                                                     \
        if (_e != cudaSuccess) {                                                     \
            set_error(std::string("CUDA: ") + cudaGetErrorString(_e) + " at " #expr); \
            return QT_ECUDA;                                                         \
        }                                                                            \
    } while (0)

struct DevBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) {
            cudaError_t e = cudaFree(p);
            if (e != cudaSuccess) return e;
            p = nullptr;
            cap = 0;
        }
        const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
        cudaError_t e = cudaMalloc(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFree(p);
        p = nullptr;
        cap = 0;
    }
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

struct HostBuf {
    void* p = nullptr;
    size_t cap = 0;
    cudaError_t ensure(size_t bytes) {
        if (bytes <= cap) return cudaSuccess;
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
        const size_t want = std::max<size_t>(bytes + bytes / 4, 256);
        cudaError_t e = cudaMallocHost(&p, want);
        if (e == cudaSuccess) cap = want;
        return e;
    }
    void release() {
        if (p) cudaFreeHost(p);
        p = nullptr;
        cap = 0;
    }
    template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

// Per-batch device + staging buffers (two of them for pipelining).
struct BatchBufs {
    DevBuf pass_start, pass_count, passes, gates, fused, cons, events, pool, records, traj_ids,
        bits, obs_out, status, counters, rho_part, blocksum, obs_part, slot_list, heap, maps;
    HostBuf h_blob, h_out;
    cudaEvent_t done = nullptr;
    cudaEvent_t prepared = nullptr;  // uploads + materialization of this batch (prep stream)
    bool inflight = false;
    // host-side bookkeeping of the batch in flight
    int nslots = 0;
    uint64_t j0 = 0;  // first trajectory ordinal of the batch
    size_t off_bits = 0, off_rec = 0, off_obs = 0, off_status = 0;
    void release() {
        for (DevBuf* b : {&pass_start, &pass_count, &passes, &gates, &fused, &cons, &events, &pool,
                          &records, &traj_ids, &bits, &obs_out, &status, &counters, &rho_part,
                          &blocksum, &obs_part, &slot_list, &heap, &maps})
            b->release();
        h_blob.release();
        h_out.release();
        if (done) cudaEventDestroy(done);
        done = nullptr;
        if (prepared) cudaEventDestroy(prepared);
        prepared = nullptr;
    }
};

}  // namespace

struct qt_ctx_s {
    int device = 0;
    cudaStream_t stream = nullptr;
    // uploads + fused-matrix materialization of the next batch overlap the
    // current batch's passes on this internal stream (ordered by events)
    cudaStream_t prep = nullptr;
    cudaEvent_t tables_ready = nullptr;
    BatchBufs bb[2];
    DevBuf vars, var_data, chans, chan_data, obs, p00, p11;
    std::vector<cudaEvent_t> prof_ev;
    std::vector<std::array<int, 5>> prof_meta;  // per timed launch: step, active slots, gates, TC-f16 gates, rho epilogues
};

namespace {

qt_status fail(qt_status st, const std::string& m) {
    set_error(m);
    return st;
}

// registers of >= 2^heap_min_lg() tiles sample through the block-sum heap (QT_HEAP_MIN_LG overrides)
int heap_min_lg() {
    static const int v = getenv("QT_HEAP_MIN_LG") ? atoi(getenv("QT_HEAP_MIN_LG")) : kHeapMinLg;
    return v;
}

// NVTX range (host timeline of the phases: planning, batch upload / launches, drain)
struct NvtxRange {
    explicit NvtxRange(const char* name) { nvtxRangePushA(name); }
    ~NvtxRange() { nvtxRangePop(); }
};

template <class F>
void parallel_for(int count, int threads, F&& fn) {
    threads = std::max(1, std::min(threads, count));
    if (threads == 1) {
        for (int i = 0; i < count; ++i) fn(i);
        return;
    }
    std::vector<std::thread> pool;
    pool.reserve(threads);
    for (int t = 0; t < threads; ++t)
        pool.emplace_back([&, t] {
            for (int i = t; i < count; i += threads) fn(i);
        });
    for (auto& th : pool) th.join();
}

template <class T>
qt_status upload(DevBuf& d, const std::vector<T>& v, cudaStream_t s) {
    QT_CK(d.ensure(std::max<size_t>(v.size() * sizeof(T), 16)));
    if (!v.empty()) QT_CK(cudaMemcpyAsync(d.p, v.data(), v.size() * sizeof(T), cudaMemcpyHostToDevice, s));
    return QT_OK;
}

// Parse Pauli strings into masks and group them by the tile they need.
qt_status parse_obs(int n, int T, int CL, int n_obs, const qt_pauli* obs, std::vector<ObsDesc>& table,
                    ObsGroups& og) {
    std::vector<ObsSpec> spec(n_obs);
    for (int k = 0; k < n_obs; ++k) {
        const qt_pauli& p = obs[k];
        if (p.nq < 0 || (p.nq > 0 && (!p.qubits || !p.paulis))) return fail(QT_EINVAL, "bad Pauli string");
        uint64_t used = 0;
        for (int i = 0; i < p.nq; ++i) {
            const int q = p.qubits[i];
            if (q < 0 || q >= n) return fail(QT_EQUBIT, "Pauli qubit out of range");
            if (used >> q & 1) return fail(QT_EQUBIT, "Pauli qubit repeated");
            used |= 1ull << q;
            switch (p.paulis[i]) {
                case 'I': break;
                case 'X': spec[k].x |= 1ull << q; break;
                case 'Y': spec[k].x |= 1ull << q; spec[k].z |= 1ull << q; spec[k].ny++; break;
                case 'Z': spec[k].z |= 1ull << q; break;
                default: return fail(QT_EINVAL, "Pauli letters must be I, X, Y or Z");
            }
        }
    }
    const uint64_t lowT = T >= 64 ? ~0ull : ((1ull << T) - 1);
    const uint64_t lowC = (1ull << std::min(CL, T)) - 1;
    og.ranges.clear();
    og.masks.clear();
    table.clear();
    // group 0: x inside the low T qubits
    std::vector<int> rest;
    og.ranges.push_back({0, 0});
    og.masks.push_back(lowT);
    for (int k = 0; k < n_obs; ++k) {
        if ((spec[k].x & ~lowT) == 0) {
            table.push_back(ObsDesc{spec[k].x, spec[k].z, spec[k].ny, k});
            og.ranges[0].second++;
        } else {
            rest.push_back(k);
        }
    }
    // strings whose X/Y part cannot fit one tile: a read-only pass over the low
    // T qubits whose CTAs read the partner tile (index ^ xmask) from HBM
    {
        const int first = (int)table.size();
        std::vector<int> left;
        for (int k : rest) {
            if (__builtin_popcountll(spec[k].x | lowC) > T) table.push_back(ObsDesc{spec[k].x, spec[k].z, spec[k].ny, k});
            else left.push_back(k);
        }
        if ((int)table.size() > first) {
            og.ranges.push_back({first, (int)table.size() - first});
            og.masks.push_back(lowT);
        }
        rest.swap(left);
    }
    while (!rest.empty()) {
        uint64_t S = lowC;
        std::vector<int> left;
        const int first = (int)table.size();
        for (int k : rest) {
            const uint64_t nm = S | spec[k].x;
            if (__builtin_popcountll(nm) <= T) {
                S = nm;
                table.push_back(ObsDesc{spec[k].x, spec[k].z, spec[k].ny, k});
            } else {
                left.push_back(k);
            }
        }
        for (int q = 0; q < n && __builtin_popcountll(S) < T; ++q) S |= 1ull << q;
        og.ranges.push_back({first, (int)table.size() - first});
        og.masks.push_back(S);
        rest.swap(left);
    }
    return QT_OK;
}

struct CallOut {
    uint64_t* bits = nullptr;
    int32_t* kraus = nullptr;
    double* obs = nullptr;
};

// Program concatenation layout (byte offsets into the host blob).
struct BlobLayout {
    size_t pass_start, pass_count, passes, gates, fused, cons, events, records, traj_ids, slot_list, end;
    size_t n_passes, n_gates, n_fused, n_cons, n_events;
    int32_t pool;
    int max_passes;
};

size_t align16(size_t x) { return (x + 15) & ~size_t(15); }

// Enqueue one batch on the stream (everything async); results land in the
// pinned h_out buffer of `B` and are copied out by finish_batch().
qt_status launch_batch(qt_ctx ctx, const Plan& P, std::vector<TrajProgram>& progs, const std::vector<uint64_t>& trajs,
                       BatchBufs& B, float2* state, int shots, uint64_t seed, int n_obs, bool want_obs,
                       bool want_bits, int obs_tables_uploaded, qt_stats* st, bool profile) {
    (void)obs_tables_uploaded;
    cudaStream_t s = ctx->stream;
    const int nslots = (int)progs.size();
    const int n = P.n;
    const int T = P.T;
    const uint32_t ntiles = 1u << (n - T);
    BlobLayout L{};
    size_t np = 0, ng = 0, nf = 0, nc = 0, ne = 0;
    int32_t pool = 0;
    int maxp = 0;
    for (auto& pg : progs) {
        np += pg.passes.size();
        ng += pg.gates.size();
        nf += pg.fused.size();
        nc += pg.cons.size();
        ne += pg.events.size();
        pool += pg.pool_size;
        maxp = std::max(maxp, (int)pg.passes.size());
    }
    size_t o = 0;
    L.pass_start = o; o = align16(o + sizeof(int32_t) * nslots);
    L.pass_count = o; o = align16(o + sizeof(int32_t) * nslots);
    L.passes = o; o = align16(o + sizeof(PassDesc) * np);
    L.gates = o; o = align16(o + sizeof(GateDesc) * ng);
    L.fused = o; o = align16(o + sizeof(FusedDesc) * nf);
    L.cons = o; o = align16(o + sizeof(ConsDesc) * nc);
    L.events = o; o = align16(o + sizeof(EventDesc) * ne);
    L.records = o; o = align16(o + sizeof(int32_t) * (size_t)nslots * std::max(P.n_recorded, 1));
    L.traj_ids = o; o = align16(o + sizeof(uint64_t) * nslots);
    // per step, the slots whose trajectory still has a pass (launch grid.y)
    std::vector<int32_t> step_off(maxp + 1, 0);
    for (int step = 0; step < maxp; ++step) {
        int act = 0;
        for (auto& pg : progs) act += step < (int)pg.passes.size();
        step_off[step + 1] = step_off[step] + act;
    }
    L.slot_list = o; o = align16(o + sizeof(PassDesc) * std::max(step_off[maxp], 1));
    L.end = o;
    QT_CK(B.h_blob.ensure(L.end));
    char* hb = B.h_blob.as<char>();
    auto* h_ps = reinterpret_cast<int32_t*>(hb + L.pass_start);
    auto* h_pc = reinterpret_cast<int32_t*>(hb + L.pass_count);
    auto* h_pass = reinterpret_cast<PassDesc*>(hb + L.passes);
    auto* h_gate = reinterpret_cast<GateDesc*>(hb + L.gates);
    auto* h_fused = reinterpret_cast<FusedDesc*>(hb + L.fused);
    auto* h_cons = reinterpret_cast<ConsDesc*>(hb + L.cons);
    auto* h_ev = reinterpret_cast<EventDesc*>(hb + L.events);
    auto* h_rec = reinterpret_cast<int32_t*>(hb + L.records);
    auto* h_tid = reinterpret_cast<uint64_t*>(hb + L.traj_ids);
    auto* h_sl = reinterpret_cast<PassDesc*>(hb + L.slot_list);
    size_t bp = 0, bg = 0, bf = 0, bc = 0, be = 0;
    int32_t bpool = 0;
    for (int b = 0; b < nslots; ++b) {
        TrajProgram& pg = progs[b];
        h_ps[b] = (int32_t)bp;
        h_pc[b] = (int32_t)pg.passes.size();
        double alg_adj = 0.0;
        for (size_t pi = 0; pi < pg.passes.size(); ++pi) {
            PassDesc pd = pg.passes[pi];
            if (pi == 0) {
                // the trajectory's first pass builds |0...0> in shared memory instead
                // of loading a zeroed state (no memset, no read; it always stores)
                if (pd.flags & kPassStore) alg_adj -= std::ldexp(1.0, n + 3);
                pd.flags |= kPassInit | kPassStore;
            }
            pd.gate_begin += (int32_t)bg;
            if (pd.event >= 0) pd.event += (int32_t)be;
            h_pass[bp++] = pd;
        }
        for (auto gd : pg.gates) {
            gd.mat_off += bpool;
            h_gate[bg++] = gd;
        }
        for (auto fd : pg.fused) {
            fd.mat_off += bpool;
            fd.cons_begin += (int32_t)bc;
            h_fused[bf++] = fd;
        }
        for (auto& c : pg.cons) h_cons[bc++] = c;
        for (auto E : pg.events) {
            E.mat_off += bpool;
            E.record = E.record >= 0 ? b * P.n_recorded + E.record : -1;
            E.slot = b;
            h_ev[be++] = E;
        }
        for (int r = 0; r < P.n_recorded; ++r) h_rec[(size_t)b * P.n_recorded + r] = pg.records[r];
        h_tid[b] = trajs[b];
        bpool += pg.pool_size;
        if (st) {
            st->passes += pg.passes.size();
            st->fused_gates += pg.gates.size();
            st->reductions += pg.events.size();
            st->channels_deferred += pg.n_deferred;
            st->channels_conventional += pg.n_conventional;
            st->alg_bytes += pg.alg_bytes + alg_adj;
            st->alg_flops += pg.alg_flops;
        }
    }
    // per-step launch arrays: this step's (rebased) pass of every active slot
    for (int step = 0, k = 0; step < maxp; ++step)
        for (int b = 0; b < nslots; ++b)
            if (step < (int)progs[b].passes.size()) {
                h_sl[k] = h_pass[h_ps[b] + step];
                h_sl[k++].slot = b;
            }
    // T = 11 (tile_pass_v3.cu): one tensor map per distinct tile layout of the batch
    // (over the batch buffer), its index in PassDesc::pad of the launch arrays
    std::vector<V3Map> v3m;
    if (P.v3) {
        std::vector<std::pair<uint64_t, int>> seen;
        for (int k = 0; k < step_off[maxp]; ++k) {
            const uint64_t m = h_sl[k].tile_mask;
            int id = -1;
            for (auto& sp : seen)
                if (sp.first == m) {
                    id = sp.second;
                    break;
                }
            if (id < 0) {
                id = (int)v3m.size();
                seen.push_back({m, id});
                v3m.emplace_back();
                if (!v3_encode_map(state, n, (uint64_t)nslots, m, &v3m.back()))
                    return fail(QT_ECUDA, "tile_pass_v3: cuTensorMapEncodeTiled failed for a tile layout");
            }
            h_sl[k].pad = id;
        }
    }
    // device buffers
    QT_CK(B.pass_start.ensure(sizeof(int32_t) * nslots));
    QT_CK(B.pass_count.ensure(sizeof(int32_t) * nslots));
    QT_CK(B.passes.ensure(sizeof(PassDesc) * std::max<size_t>(np, 1)));
    QT_CK(B.gates.ensure(sizeof(GateDesc) * std::max<size_t>(ng, 1)));
    QT_CK(B.fused.ensure(sizeof(FusedDesc) * std::max<size_t>(nf, 1)));
    QT_CK(B.cons.ensure(sizeof(ConsDesc) * std::max<size_t>(nc, 1)));
    QT_CK(B.events.ensure(sizeof(EventDesc) * std::max<size_t>(ne, 1)));
    QT_CK(B.records.ensure(sizeof(int32_t) * (size_t)nslots * std::max(P.n_recorded, 1)));
    QT_CK(B.traj_ids.ensure(sizeof(uint64_t) * nslots));
    QT_CK(B.slot_list.ensure(sizeof(PassDesc) * std::max(step_off[maxp], 1)));
    QT_CK(B.pool.ensure(sizeof(float2) * std::max<int32_t>(pool, 2)));
    QT_CK(B.status.ensure(sizeof(int32_t) * nslots));
    QT_CK(B.counters.ensure(sizeof(int32_t) * nslots));
    const int rd = P.max_chan_d;  // conventional mode reduces every channel (q <= 6)
    const int rho_stride = 2 * rd * rd;
    QT_CK(B.rho_part.ensure(sizeof(double) * (size_t)nslots * ntiles * rho_stride));
    QT_CK(B.blocksum.ensure(sizeof(double) * (size_t)nslots * ntiles));
    QT_CK(B.obs_part.ensure(sizeof(double) * (size_t)nslots * ntiles * std::max(n_obs, 1)));
    QT_CK(B.obs_out.ensure(sizeof(double) * (size_t)nslots * std::max(n_obs, 1)));
    QT_CK(B.bits.ensure(sizeof(uint64_t) * (size_t)nslots * std::max(shots, 1)));
    // one contiguous H2D per region, on the prep stream (the previous user of
    // these buffers finished: finish_batch waited on B.done)
    cudaStream_t ps = ctx->prep;
    auto h2d = [&](DevBuf& d, size_t off, size_t bytes) -> qt_status {
        if (bytes) QT_CK(cudaMemcpyAsync(d.p, hb + off, bytes, cudaMemcpyHostToDevice, ps));
        return QT_OK;
    };
    qt_status e;
    if ((e = h2d(B.pass_start, L.pass_start, sizeof(int32_t) * nslots)) != QT_OK) return e;
    if ((e = h2d(B.pass_count, L.pass_count, sizeof(int32_t) * nslots)) != QT_OK) return e;
    if ((e = h2d(B.passes, L.passes, sizeof(PassDesc) * np)) != QT_OK) return e;
    if ((e = h2d(B.gates, L.gates, sizeof(GateDesc) * ng)) != QT_OK) return e;
    if ((e = h2d(B.fused, L.fused, sizeof(FusedDesc) * nf)) != QT_OK) return e;
    if ((e = h2d(B.cons, L.cons, sizeof(ConsDesc) * nc)) != QT_OK) return e;
    if ((e = h2d(B.events, L.events, sizeof(EventDesc) * ne)) != QT_OK) return e;
    if ((e = h2d(B.records, L.records, sizeof(int32_t) * (size_t)nslots * P.n_recorded)) != QT_OK) return e;
    if ((e = h2d(B.traj_ids, L.traj_ids, sizeof(uint64_t) * nslots)) != QT_OK) return e;
    if ((e = h2d(B.slot_list, L.slot_list, sizeof(PassDesc) * step_off[maxp])) != QT_OK) return e;
    if (!v3m.empty()) {
        QT_CK(B.maps.ensure(sizeof(V3Map) * v3m.size()));
        QT_CK(cudaMemcpyAsync(B.maps.p, v3m.data(), sizeof(V3Map) * v3m.size(), cudaMemcpyHostToDevice, ps));
        QT_CK(cudaStreamSynchronize(ps));  // v3m is a local
    }
    QT_CK(cudaMemsetAsync(B.status.p, 0, sizeof(int32_t) * nslots, ps));
    QT_CK(cudaMemsetAsync(B.counters.p, 0, sizeof(int32_t) * nslots, ps));
    QT_CK(launch_materialize(B.fused.as<FusedDesc>(), (int)nf, P.tc ? P.tc_k : P.R, B.cons.as<ConsDesc>(),
                             ctx->vars.as<VarDesc>(),
                             ctx->var_data.as<double>(), B.pool.as<float2>(), ps));
    if (!B.prepared) QT_CK(cudaEventCreateWithFlags(&B.prepared, cudaEventDisableTiming));
    QT_CK(cudaEventRecord(B.prepared, ps));
    QT_CK(cudaStreamWaitEvent(s, B.prepared, 0));
    // |0...0> in every slot: built by the first pass of each trajectory (kPassInit)
    uint64_t launches = (nf > 0);
    TileArgs A;
    A.state = state;
    A.n = n;
    A.T = T;
    A.passes = B.passes.as<PassDesc>();
    A.pass_start = B.pass_start.as<int32_t>();
    A.pass_count = B.pass_count.as<int32_t>();
    A.gates = B.gates.as<GateDesc>();
    A.pool = B.pool.as<float2>();
    A.events = B.events.as<EventDesc>();
    A.chans = ctx->chans.as<ChanDesc>();
    A.chan_data = ctx->chan_data.as<double>();
    A.rho_part = B.rho_part.as<double>();
    A.rho_stride = rho_stride;
    A.counters = B.counters.as<int32_t>();
    A.records = B.records.as<int32_t>();
    A.status = B.status.as<int32_t>();
    A.blocksum = B.blocksum.as<double>();
    A.obs_part = B.obs_part.as<double>();
    A.n_obs = n_obs;
    A.obs = ctx->obs.as<ObsDesc>();
    A.v3maps = P.v3 ? B.maps.p : nullptr;
    for (int step = 0; step < maxp; ++step) {
        const int act = step_off[step + 1] - step_off[step];
        A.step_passes = B.slot_list.as<PassDesc>() + step_off[step];
        if (profile) {
            cudaEvent_t e0, e1;
            QT_CK(cudaEventCreate(&e0));
            QT_CK(cudaEventCreate(&e1));
            QT_CK(cudaEventRecord(e0, s));
            QT_CK(launch_tile_pass(A, P.R, P.tc ? P.tc_k : 0, step, ntiles, act, s));
            QT_CK(cudaEventRecord(e1, s));
            ctx->prof_ev.push_back(e0);
            ctx->prof_ev.push_back(e1);
            std::array<int, 5> m{step, 0, 0, 0, 0};
            for (auto& pg : progs)
                if (step < (int)pg.passes.size()) {
                    const PassDesc& pd = pg.passes[step];
                    ++m[1];
                    m[2] += pd.gate_count;
                    m[4] += (pd.flags & kPassRho) != 0;
                    for (int g = 0; g < pd.gate_count; ++g) m[3] += (pg.gates[pd.gate_begin + g].k & kGateF16) != 0;
                }
            ctx->prof_meta.push_back(m);
        } else {
            QT_CK(launch_tile_pass(A, P.R, P.tc ? P.tc_k : 0, step, ntiles, act, s));
        }
        ++launches;
    }
    if (want_obs && n_obs > 0) {
        QT_CK(launch_finalize_obs(B.blocksum.as<double>(), B.obs_part.as<double>(), (int)ntiles, n_obs, nslots,
                                  B.obs_out.as<double>(), nullptr, s));
        ++launches;
        if (const char* dump = std::getenv("QT_DUMP_PARTIALS")) {  // diagnostics: block sums + observable partials
            std::vector<double> hb((size_t)nslots * ntiles), ho((size_t)nslots * ntiles * n_obs);
            cudaMemcpyAsync(hb.data(), B.blocksum.p, hb.size() * 8, cudaMemcpyDeviceToHost, s);
            cudaMemcpyAsync(ho.data(), B.obs_part.p, ho.size() * 8, cudaMemcpyDeviceToHost, s);
            cudaStreamSynchronize(s);
            if (FILE* f = std::fopen(dump, "wb")) {
                std::fwrite(hb.data(), 8, hb.size(), f);
                std::fwrite(ho.data(), 8, ho.size(), f);
                std::fclose(f);
            }
        }
    }
    if (want_bits && shots > 0) {
        double* heap = nullptr;
        if (n - T >= heap_min_lg()) {
            QT_CK(B.heap.ensure(sizeof(double) * 2 * (size_t)nslots * ntiles));
            heap = B.heap.as<double>();
        }
        QT_CK(launch_sample(state, n, T, B.blocksum.as<double>(), nslots, shots, seed, B.traj_ids.as<uint64_t>(),
                            P.has_p00 ? ctx->p00.as<double>() : nullptr, P.has_p11 ? ctx->p11.as<double>() : nullptr,
                            B.bits.as<uint64_t>(), s, 0, nullptr, heap));
        ++launches;
    }
    if (st) st->launches += launches;
    // D2H of the results into the pinned output blob
    B.off_bits = 0;
    B.off_rec = align16(B.off_bits + sizeof(uint64_t) * (size_t)nslots * std::max(shots, 0));
    B.off_obs = align16(B.off_rec + sizeof(int32_t) * (size_t)nslots * P.n_recorded);
    B.off_status = align16(B.off_obs + sizeof(double) * (size_t)nslots * std::max(n_obs, 0));
    const size_t out_bytes = align16(B.off_status + sizeof(int32_t) * nslots);
    QT_CK(B.h_out.ensure(out_bytes));
    if (st) {
        st->h2d_bytes += L.end;
        st->d2h_bytes += (want_bits && shots > 0 ? sizeof(uint64_t) * (size_t)nslots * shots : 0) +
                         sizeof(int32_t) * (size_t)nslots * (P.n_recorded + 1) +
                         (want_obs ? sizeof(double) * (size_t)nslots * n_obs : 0);
    }
    char* ho = B.h_out.as<char>();
    if (want_bits && shots > 0)
        QT_CK(cudaMemcpyAsync(ho + B.off_bits, B.bits.p, sizeof(uint64_t) * (size_t)nslots * shots,
                              cudaMemcpyDeviceToHost, s));
    if (P.n_recorded > 0)
        QT_CK(cudaMemcpyAsync(ho + B.off_rec, B.records.p, sizeof(int32_t) * (size_t)nslots * P.n_recorded,
                              cudaMemcpyDeviceToHost, s));
    if (want_obs && n_obs > 0)
        QT_CK(cudaMemcpyAsync(ho + B.off_obs, B.obs_out.p, sizeof(double) * (size_t)nslots * n_obs,
                              cudaMemcpyDeviceToHost, s));
    QT_CK(cudaMemcpyAsync(ho + B.off_status, B.status.p, sizeof(int32_t) * nslots, cudaMemcpyDeviceToHost, s));
    if (!B.done) QT_CK(cudaEventCreateWithFlags(&B.done, cudaEventDisableTiming));
    QT_CK(cudaEventRecord(B.done, s));
    B.inflight = true;
    B.nslots = nslots;
    return QT_OK;
}

qt_status finish_batch(BatchBufs& B, const Plan& P, int shots, int n_obs, const CallOut& out) {
    if (!B.inflight) return QT_OK;
    QT_CK(cudaEventSynchronize(B.done));
    B.inflight = false;
    const char* ho = B.h_out.as<char>();
    const int ns = B.nslots;
    const auto* status = reinterpret_cast<const int32_t*>(ho + B.off_status);
    for (int b = 0; b < ns; ++b)
        if (status[b] != 0) {
            const int code = status[b];
            set_error("device status " + std::to_string(code) + " in trajectory slot " + std::to_string(b) +
                      (code == -9 ? " (Alg. 2 fall-through residual > 1e-6)" : ""));
            return (qt_status)code;
        }
    if (out.bits && shots > 0)
        std::memcpy(out.bits + B.j0 * shots, ho + B.off_bits, sizeof(uint64_t) * (size_t)ns * shots);
    if (out.kraus && P.n_recorded > 0)
        std::memcpy(out.kraus + B.j0 * P.n_recorded, ho + B.off_rec, sizeof(int32_t) * (size_t)ns * P.n_recorded);
    if (out.obs && n_obs > 0)
        std::memcpy(out.obs + B.j0 * n_obs, ho + B.off_obs, sizeof(double) * (size_t)ns * n_obs);
    return QT_OK;
}

qt_status upload_plan_tables(qt_ctx ctx, const Plan& P, const std::vector<ObsDesc>& obs_table) {
    cudaStream_t s = ctx->stream;
    qt_status e;
    if ((e = upload(ctx->vars, P.var_desc, s)) != QT_OK) return e;
    if ((e = upload(ctx->var_data, P.var_data, s)) != QT_OK) return e;
    if ((e = upload(ctx->chans, P.chans, s)) != QT_OK) return e;
    if ((e = upload(ctx->chan_data, P.chan_data, s)) != QT_OK) return e;
    if ((e = upload(ctx->obs, obs_table, s)) != QT_OK) return e;
    if (P.has_p00 && (e = upload(ctx->p00, P.p00, s)) != QT_OK) return e;
    if (P.has_p11 && (e = upload(ctx->p11, P.p11, s)) != QT_OK) return e;
    return QT_OK;
}

}  // namespace

extern "C" {

qt_status qt_ctx_create(int device, void* cuda_stream, qt_ctx* out) {
    if (!out) return fail(QT_EINVAL, "out is NULL");
    int count = 0;
    cudaError_t e = cudaGetDeviceCount(&count);
    if (e != cudaSuccess || count == 0)
        return fail(QT_ECUDA, std::string("no CUDA device: ") + cudaGetErrorString(e));
    if (device < 0 || device >= count) return fail(QT_EINVAL, "device ordinal out of range");
    QT_CK(cudaSetDevice(device));
    cudaDeviceProp prop;
    QT_CK(cudaGetDeviceProperties(&prop, device));
    if (prop.major != 10) return fail(QT_ECUDA, "libqtraj is built for sm_100a (B200) only");
    auto* c = new (std::nothrow) qt_ctx_s();
    if (!c) return fail(QT_EOOM, "host allocation failed");
    c->device = device;
    c->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    QT_CK(cudaStreamCreateWithFlags(&c->prep, cudaStreamNonBlocking));
    QT_CK(cudaEventCreateWithFlags(&c->tables_ready, cudaEventDisableTiming));
    *out = c;
    return QT_OK;
}

qt_status qt_ctx_set_stream(qt_ctx ctx, void* cuda_stream) {
    if (!ctx) return fail(QT_EINVAL, "NULL ctx");
    ctx->stream = reinterpret_cast<cudaStream_t>(cuda_stream);
    return QT_OK;
}

void qt_ctx_destroy(qt_ctx ctx) {
    if (!ctx) return;
    cudaSetDevice(ctx->device);
    cudaStreamSynchronize(ctx->stream);
    for (auto& b : ctx->bb) b.release();
    for (DevBuf* d : {&ctx->vars, &ctx->var_data, &ctx->chans, &ctx->chan_data, &ctx->obs, &ctx->p00, &ctx->p11})
        d->release();
    for (auto ev : ctx->prof_ev) cudaEventDestroy(ev);
    if (ctx->prep) {
        cudaStreamSynchronize(ctx->prep);
        cudaStreamDestroy(ctx->prep);
    }
    if (ctx->tables_ready) cudaEventDestroy(ctx->tables_ready);
    delete ctx;
}

qt_status qt_run_trajectories(qt_ctx ctx, qt_plan plan, const qt_run_opts* opts, int n_obs, const qt_pauli* obs,
                              void* state_dev, size_t state_bytes, uint64_t* out_bits, int32_t* out_kraus,
                              double* out_obs, qt_stats* out_stats) {
    NvtxRange nvtx_call("qt_run_trajectories");
    if (!ctx || !plan || !opts || !state_dev) return fail(QT_EINVAL, "NULL argument");
    if (n_obs < 0 || (n_obs > 0 && !obs)) return fail(QT_EINVAL, "bad observables");
    if (opts->mode != 0 && opts->mode != 1) return fail(QT_EINVAL, "mode must be 0 (delayed) or 1 (conventional)");
    if (opts->shots_per_traj < 0) return fail(QT_EINVAL, "shots_per_traj < 0");
    // conventional mode reduces every channel: channels on 4..6 qubits need the
    // CUDA-core kernel (its device-chosen operators hold 2^6 amplitudes per thread)
    Plan fallback;
    const Plan* Pp = &plan_of(plan);
    if (opts->mode == 1 && Pp->max_chan_d > 8 && Pp->tc) {
        fallback = *Pp;
        cuda_core_plan(fallback);
        Pp = &fallback;
    }
    const Plan& P = *Pp;
    QT_CK(cudaSetDevice(ctx->device));
    const size_t per = sizeof(float2) << P.n;
    const size_t max_slots = state_bytes / per;
    if (max_slots < 1) return fail(QT_EOOM, "state buffer smaller than one 2^n complex64 state");
    int batch = opts->batch > 0 ? opts->batch : 256;
    batch = (int)std::min<size_t>((size_t)batch, max_slots);
    batch = std::min(batch, 65535);
    // T = 11 (tile_pass_v3.cu): TMA rest coordinates are int32 units of 16 amplitudes over
    // the whole batch buffer
    if (P.v3) batch = (int)std::min<int64_t>((int64_t)batch, std::max<int64_t>(1, (int64_t(1) << 31) >> (P.n - 4)));
    const uint64_t stride = opts->traj_stride ? opts->traj_stride : 1;
    const int shots = opts->shots_per_traj;
    int threads = opts->host_threads > 0 ? opts->host_threads : (int)std::thread::hardware_concurrency();
    threads = std::max(threads, 1);
    qt_stats st{};
    std::vector<ObsDesc> obs_table;
    ObsGroups og;
    qt_status e = parse_obs(P.n, P.T, P.CL, n_obs, obs, obs_table, og);
    if (e != QT_OK) return e;
    cudaStream_t s = ctx->stream;
    cudaEvent_t t0, t1;
    QT_CK(cudaEventCreate(&t0));
    QT_CK(cudaEventCreate(&t1));
    QT_CK(cudaEventRecord(t0, s));
    if ((e = upload_plan_tables(ctx, P, obs_table)) != QT_OK) return e;
    QT_CK(cudaEventRecord(ctx->tables_ready, s));  // materialization (prep stream) reads the tables
    QT_CK(cudaStreamWaitEvent(ctx->prep, ctx->tables_ready, 0));
    st.h2d_bytes += sizeof(VarDesc) * P.var_desc.size() + sizeof(double) * P.var_data.size() +
                    sizeof(ChanDesc) * P.chans.size() + sizeof(double) * P.chan_data.size() +
                    sizeof(ObsDesc) * obs_table.size() + sizeof(double) * (P.p00.size() + P.p11.size());
    for (auto ev : ctx->prof_ev) cudaEventDestroy(ev);
    ctx->prof_ev.clear();
    ctx->prof_meta.clear();
    const CallOut out{out_bits, out_kraus, out_obs};
    double plan_ms = 0;
    float2* state = reinterpret_cast<float2*>(state_dev);
    // Two batch slots alternate; the state buffer is shared, so batch i+1's
    // device work is stream-ordered after batch i (same stream) while its host
    // planning overlaps batch i's device execution.
    std::vector<TrajProgram> progs;
    std::vector<uint64_t> trajs;
    int which = 0;
    qt_status status = QT_OK;
    for (uint64_t j0 = 0; j0 < opts->traj_count && status == QT_OK; j0 += (uint64_t)batch) {
        const int ns = (int)std::min<uint64_t>((uint64_t)batch, opts->traj_count - j0);
        progs.resize(ns);  // plan_trajectory resets a program keeping its capacity
        trajs.resize(ns);
        for (int b = 0; b < ns; ++b) trajs[b] = opts->traj_begin + (j0 + b) * stride;
        std::vector<qt_status> pst(ns, QT_OK);
        const auto h0 = std::chrono::steady_clock::now();
        {
            NvtxRange r("qt: plan batch (Alg. 2 first loop + fuser)");
            parallel_for(ns, threads,
                         [&](int b) { pst[b] = plan_trajectory(P, opts->seed, trajs[b], og, progs[b], opts->mode); });
        }
        plan_ms += std::chrono::duration<double, std::milli>(std::chrono::steady_clock::now() - h0).count();
        for (int b = 0; b < ns; ++b)
            if (pst[b] != QT_OK) status = pst[b];
        if (status != QT_OK) break;
        BatchBufs& B = ctx->bb[which];
        // the slot's previous batch must be finished before its buffers are reused
        {
            NvtxRange r("qt: drain previous batch");
            if ((status = finish_batch(B, P, shots, n_obs, out)) != QT_OK) break;
        }
        B.j0 = j0;
        NvtxRange r("qt: upload + launch batch");
        status = launch_batch(ctx, P, progs, trajs, B, state, shots, opts->seed, n_obs, n_obs > 0, shots > 0, 1, &st,
                              opts->profile != 0);
        which ^= 1;
    }
    for (auto& B : ctx->bb) {
        qt_status e2 = finish_batch(B, P, shots, n_obs, out);
        if (status == QT_OK) status = e2;
    }
    QT_CK(cudaEventRecord(t1, s));
    QT_CK(cudaEventSynchronize(t1));
    float ms = 0;
    cudaEventElapsedTime(&ms, t0, t1);
    cudaEventDestroy(t0);
    cudaEventDestroy(t1);
    if (opts->profile) {
        double pm = 0;
        for (size_t i = 0; i + 1 < ctx->prof_ev.size(); i += 2) {
            float x = 0;
            cudaEventElapsedTime(&x, ctx->prof_ev[i], ctx->prof_ev[i + 1]);
            pm += x;
        }
        st.pass_kernel_ms = pm;
        st.pass_launches = ctx->prof_ev.size() / 2;
        // diagnostics: per-launch times and pass composition
        if (const char* dump = std::getenv("QT_PROFILE_DUMP")) {
            if (FILE* f = std::fopen(dump, "a")) {
                for (size_t i = 0; i + 1 < ctx->prof_ev.size() && i / 2 < ctx->prof_meta.size(); i += 2) {
                    float x = 0;
                    cudaEventElapsedTime(&x, ctx->prof_ev[i], ctx->prof_ev[i + 1]);
                    const auto& m = ctx->prof_meta[i / 2];
                    std::fprintf(f, "%d %d %d %d %d %.4f\n", m[0], m[1], m[2], m[3], m[4], x);
                }
                std::fclose(f);
            }
        }
    }
    st.trajectories = opts->traj_count;
    st.plan_ms = plan_ms;
    st.device_ms = ms;
    if (out_stats) *out_stats = st;
    return status;
}

// ---- stand-alone state operations -----------------------------------------

// Extra inputs/outputs of the stand-alone path (distributed-state mode).
struct SingleExtras {
    double* out_norm = nullptr;        // <psi|psi> of the state (with out_obs)
    int n_rng = 0;                     // qubits of the whole register for the SAMPLE ordinals
    const int32_t* shot_ids = nullptr; // host: shot ordinal of each sampled shot
};

static qt_status run_single(qt_ctx ctx, qt_plan plan, float2* state, const ObsGroups& og,
                            const std::vector<ObsDesc>& obs_table, int n_obs, int shots, uint64_t seed,
                            uint64_t traj, uint64_t* out_bits, double* out_obs, int repeats, double* kernel_ms,
                            bool zero_state, const SingleExtras* ex = nullptr) {
    const Plan& P = plan_of(plan);
    if (P.v3) return fail(QT_EINVAL, "plans with tile_bits = 11 run through qt_run_trajectories only");
    QT_CK(cudaSetDevice(ctx->device));
    qt_status e = upload_plan_tables(ctx, P, obs_table);
    if (e != QT_OK) return e;
    std::vector<TrajProgram> progs(1);
    if ((e = plan_trajectory(P, seed, traj, og, progs[0])) != QT_OK) return e;
    std::vector<uint64_t> trajs{traj};
    BatchBufs& B = ctx->bb[0];
    if ((e = finish_batch(ctx->bb[1], P, 0, 0, CallOut{})) != QT_OK) return e;
    if ((e = finish_batch(B, P, 0, 0, CallOut{})) != QT_OK) return e;
    (void)zero_state;
    // launch_batch zero-initializes the state; stand-alone operations must not,
    // so drive the pieces directly.
    cudaStream_t s = ctx->stream;
    TrajProgram& pg = progs[0];
    const int n = P.n, T = P.T;
    const uint32_t ntiles = 1u << (n - T);
    qt_status r;
    if ((r = upload(B.passes, pg.passes, s)) != QT_OK) return r;
    if ((r = upload(B.gates, pg.gates, s)) != QT_OK) return r;
    if ((r = upload(B.fused, pg.fused, s)) != QT_OK) return r;
    if ((r = upload(B.cons, pg.cons, s)) != QT_OK) return r;
    std::vector<int32_t> ps{0}, pc{(int32_t)pg.passes.size()};
    if ((r = upload(B.pass_start, ps, s)) != QT_OK) return r;
    if ((r = upload(B.pass_count, pc, s)) != QT_OK) return r;
    if ((r = upload(B.traj_ids, trajs, s)) != QT_OK) return r;
    QT_CK(B.pool.ensure(sizeof(float2) * std::max<int32_t>(pg.pool_size, 2)));
    QT_CK(B.status.ensure(sizeof(int32_t)));
    QT_CK(B.counters.ensure(sizeof(int32_t)));
    QT_CK(B.rho_part.ensure(sizeof(double) * ntiles * 8));
    QT_CK(B.blocksum.ensure(sizeof(double) * ntiles));
    QT_CK(B.obs_part.ensure(sizeof(double) * (size_t)ntiles * std::max(n_obs, 1)));
    QT_CK(B.obs_out.ensure(sizeof(double) * std::max(n_obs, 1)));
    QT_CK(B.bits.ensure(sizeof(uint64_t) * std::max(shots, 1)));
    QT_CK(B.events.ensure(16));
    QT_CK(B.records.ensure(16));
    QT_CK(cudaMemsetAsync(B.status.p, 0, sizeof(int32_t), s));
    QT_CK(cudaMemsetAsync(B.counters.p, 0, sizeof(int32_t), s));
    QT_CK(launch_materialize(B.fused.as<FusedDesc>(), (int)pg.fused.size(), P.tc ? P.tc_k : P.R, B.cons.as<ConsDesc>(),
                             ctx->vars.as<VarDesc>(), ctx->var_data.as<double>(), B.pool.as<float2>(), s));
    TileArgs A{};
    A.state = state;
    A.n = n;
    A.T = T;
    A.passes = B.passes.as<PassDesc>();
    A.pass_start = B.pass_start.as<int32_t>();
    A.pass_count = B.pass_count.as<int32_t>();
    A.gates = B.gates.as<GateDesc>();
    A.pool = B.pool.as<float2>();
    A.events = B.events.as<EventDesc>();
    A.chans = ctx->chans.as<ChanDesc>();
    A.chan_data = ctx->chan_data.as<double>();
    A.rho_part = B.rho_part.as<double>();
    A.rho_stride = 8;
    A.counters = B.counters.as<int32_t>();
    A.records = B.records.as<int32_t>();
    A.status = B.status.as<int32_t>();
    A.blocksum = B.blocksum.as<double>();
    A.obs_part = B.obs_part.as<double>();
    A.n_obs = n_obs;
    A.obs = ctx->obs.as<ObsDesc>();
    const int np = (int)pg.passes.size();
    cudaEvent_t e0 = nullptr, e1 = nullptr;
    if (kernel_ms) {
        QT_CK(cudaEventCreate(&e0));
        QT_CK(cudaEventCreate(&e1));
    }
    for (int rep = 0; rep < std::max(repeats, 1); ++rep) {
        if (kernel_ms && rep == 1) QT_CK(cudaEventRecord(e0, s));  // rep 0 = warm-up
        for (int step = 0; step < np; ++step) {
            A.step_passes = B.passes.as<PassDesc>() + step;  // one slot: its pass of this step (slot 0)
            QT_CK(launch_tile_pass(A, P.R, P.tc ? P.tc_k : 0, step, ntiles, 1, s));
        }
    }
    if (kernel_ms) {
        if (repeats <= 1) QT_CK(cudaEventRecord(e0, s));
        QT_CK(cudaEventRecord(e1, s));
    }
    const bool want_norm = ex && ex->out_norm;
    if ((out_obs && n_obs > 0) || want_norm)
        QT_CK(launch_finalize_obs(B.blocksum.as<double>(), B.obs_part.as<double>(), (int)ntiles, n_obs, 1,
                                  B.obs_out.as<double>(), B.records.as<double>() /* 16 B scratch: norm */, s));
    int32_t* dshots = nullptr;
    if (out_bits && shots > 0) {
        if (ex && ex->shot_ids) {
            QT_CK(B.counters.ensure(sizeof(int32_t) * std::max(shots, 1)));
            QT_CK(cudaMemcpyAsync(B.counters.p, ex->shot_ids, sizeof(int32_t) * shots, cudaMemcpyHostToDevice, s));
            dshots = B.counters.as<int32_t>();
        }
        double* heap = nullptr;
        if (n - T >= heap_min_lg()) {
            QT_CK(B.heap.ensure(sizeof(double) * 2 * (size_t)ntiles));
            heap = B.heap.as<double>();
        }
        QT_CK(launch_sample(state, n, T, B.blocksum.as<double>(), 1, shots, seed, B.traj_ids.as<uint64_t>(), nullptr,
                            nullptr, B.bits.as<uint64_t>(), s, ex ? ex->n_rng : 0, dshots, heap));
    }
    std::vector<double> obs_host(std::max(n_obs, 1));
    if (out_obs && n_obs > 0)
        QT_CK(cudaMemcpyAsync(obs_host.data(), B.obs_out.p, sizeof(double) * n_obs, cudaMemcpyDeviceToHost, s));
    if (want_norm) QT_CK(cudaMemcpyAsync(ex->out_norm, B.records.p, sizeof(double), cudaMemcpyDeviceToHost, s));
    if (out_bits && shots > 0)
        QT_CK(cudaMemcpyAsync(out_bits, B.bits.p, sizeof(uint64_t) * shots, cudaMemcpyDeviceToHost, s));
    QT_CK(cudaStreamSynchronize(s));
    if (out_obs && n_obs > 0)
        for (int k = 0; k < n_obs; ++k) out_obs[k] = obs_host[k];  // finalize writes column = ObsDesc::slot
    if (kernel_ms) {
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        *kernel_ms = repeats > 1 ? ms / (repeats - 1) : ms;
        cudaEventDestroy(e0);
        cudaEventDestroy(e1);
    }
    return QT_OK;
}

qt_status qt_apply_gate_ex(qt_ctx ctx, void* state_dev, int n, int nq, const int* qubits, const double* U,
                           int repeats, double* kernel_ms) {
    NvtxRange nvtx_call("qt_apply_gate");
    if (!ctx || !state_dev) return fail(QT_EINVAL, "NULL argument");
    qt_circuit c = nullptr;
    qt_status e = qt_circuit_create(n, &c);
    if (e != QT_OK) return e;
    if ((e = qt_add_gate(c, 0, nq, qubits, U)) != QT_OK) {
        qt_circuit_destroy(c);
        return e;
    }
    // the streaming single-gate kernel (TMA tiles, tensor cores) when the register holds
    // its tiles; QT_GATE_STREAM=0 selects the trajectory kernels for A/B runs
    static const bool stream_off = getenv("QT_GATE_STREAM") && atoi(getenv("QT_GATE_STREAM")) == 0;
    if (!stream_off) {
        const HostOp* op = circuit_op(c, 0);
        cudaError_t ce = gate_stream_apply(ctx->stream, state_dev, n, op->nq, op->q, op->mats.data(), repeats, kernel_ms);
        if (ce != cudaErrorNotSupported) {
            qt_circuit_destroy(c);
            if (ce != cudaSuccess) return fail(QT_ECUDA, std::string("gate_stream: ") + cudaGetErrorString(ce));
            return QT_OK;
        }
        cudaGetLastError();
    }
    qt_fuse_opts o{};
    o.max_fused = std::max(nq, 2);
    // one fused gate per HBM pass: the per-tile kernel (12-qubit tiles) streams these faster
    // than the persistent kernel, whose strength is long in-TMEM gate chains
    if (n >= 12) o.tile_bits = 12;
    qt_plan p = nullptr;
    e = qt_fuse_ex(c, &o, &p);
    qt_circuit_destroy(c);
    if (e != QT_OK) return e;
    ObsGroups og;
    og.final_pass = false;
    e = run_single(ctx, p, reinterpret_cast<float2*>(state_dev), og, {}, 0, 0, 0, 0, nullptr, nullptr, repeats,
                   kernel_ms, false);
    qt_plan_destroy(p);
    return e;
}

qt_status qt_apply_gate(qt_ctx ctx, void* state_dev, int n, int nq, const int* qubits, const double* U) {
    return qt_apply_gate_ex(ctx, state_dev, n, nq, qubits, U, 1, nullptr);
}

qt_status qt_plan_info(qt_plan plan, uint64_t seed, uint64_t traj, int64_t* out) {
    if (!plan || !out) return fail(QT_EINVAL, "NULL argument");
    const Plan& P = plan_of(plan);
    ObsGroups og;
    og.ranges.push_back({0, 0});
    og.masks.push_back(0);
    TrajProgram pg;
    qt_status e = plan_trajectory(P, seed, traj, og, pg);
    if (e != QT_OK) return e;
    out[0] = (int64_t)pg.passes.size();
    out[1] = (int64_t)pg.gates.size();
    out[2] = (int64_t)pg.events.size();
    out[3] = (int64_t)pg.n_deferred;
    out[4] = (int64_t)pg.n_conventional;
    out[5] = (int64_t)pg.pool_size;
    out[6] = (int64_t)pg.alg_bytes;
    out[7] = (int64_t)pg.cons.size();
    out[8] = P.T;
    out[9] = P.v3 ? 11 : (P.v2 ? 13 : (P.tc ? P.tc_k : 0));
    return QT_OK;
}

// Diagnostic (undeclared): host planning cost -- plans trajectories traj0 .. traj0 + count - 1
// on one thread into one reused program (as the runtime's per-slot programs are reused)
// and returns the seconds spent.
extern "C" qt_status qt_plan_bench(qt_plan plan, uint64_t seed, uint64_t traj0, int count, double* seconds) {
    if (!plan || !seconds || count < 0) return fail(QT_EINVAL, "bad argument");
    const Plan& P = plan_of(plan);
    ObsGroups og;
    og.ranges.push_back({0, 0});
    og.masks.push_back(0);
    TrajProgram pg;
    const auto t0 = std::chrono::steady_clock::now();
    for (int j = 0; j < count; ++j) {
        const qt_status e = plan_trajectory(P, seed, traj0 + (uint64_t)j, og, pg);
        if (e != QT_OK) return e;
    }
    *seconds = std::chrono::duration<double>(std::chrono::steady_clock::now() - t0).count();
    return QT_OK;
}

static qt_status read_only_plan(int n, qt_plan* p) {
    qt_circuit c = nullptr;
    qt_status e = qt_circuit_create(n, &c);
    if (e != QT_OK) return e;
    e = qt_fuse(c, 4, p);
    qt_circuit_destroy(c);
    return e;
}

qt_status qt_sample_bitstrings(qt_ctx ctx, const void* state_dev, int n, uint64_t seed, uint64_t traj, int shots,
                               uint64_t* out) {
    if (!ctx || !state_dev || (!out && shots > 0) || shots < 0) return fail(QT_EINVAL, "bad argument");
    qt_plan p = nullptr;
    qt_status e = read_only_plan(n, &p);
    if (e != QT_OK) return e;
    ObsGroups og;
    og.ranges.push_back({0, 0});
    og.masks.push_back(0);
    e = run_single(ctx, p, const_cast<float2*>(reinterpret_cast<const float2*>(state_dev)), og, {}, 0, shots, seed,
                   traj, out, nullptr, 1, nullptr, false);
    qt_plan_destroy(p);
    return e;
}

qt_status qt_expectation_value(qt_ctx ctx, const void* state_dev, int n, int n_obs, const qt_pauli* obs,
                               double* out) {
    if (!ctx || !state_dev || (n_obs > 0 && (!obs || !out))) return fail(QT_EINVAL, "bad argument");
    qt_plan p = nullptr;
    qt_status e = read_only_plan(n, &p);
    if (e != QT_OK) return e;
    const Plan& P = plan_of(p);
    std::vector<ObsDesc> table;
    ObsGroups og;
    if ((e = parse_obs(n, P.T, P.CL, n_obs, obs, table, og)) == QT_OK)
        e = run_single(ctx, p, const_cast<float2*>(reinterpret_cast<const float2*>(state_dev)), og, table, n_obs, 0,
                       0, 0, nullptr, out, 1, nullptr, false);
    qt_plan_destroy(p);
    return e;
}

// ---- building blocks of the distributed-state mode -------------------------

qt_status qt_permute_qubits(qt_ctx ctx, const void* src_dev, void* dst_dev, int n, const int* perm) {
    if (!ctx || !src_dev || !dst_dev || !perm || src_dev == dst_dev) return fail(QT_EINVAL, "bad argument");
    if (n < 1 || n > 40) return fail(QT_EINVAL, "qt_permute_qubits: 1 <= n <= 40");
    uint64_t seen = 0;
    for (int b = 0; b < n; ++b) {
        if (perm[b] < 0 || perm[b] >= n || ((seen >> perm[b]) & 1ull)) return fail(QT_EQUBIT, "not a permutation");
        seen |= 1ull << perm[b];
    }
    QT_CK(cudaSetDevice(ctx->device));
    QT_CK(launch_permute_qubits(reinterpret_cast<const float2*>(src_dev), reinterpret_cast<float2*>(dst_dev), n, perm,
                                ctx->stream));
    return QT_OK;
}

qt_status qt_apply_plan(qt_ctx ctx, qt_plan plan, void* state_dev, size_t state_bytes) {
    if (!ctx || !plan || !state_dev) return fail(QT_EINVAL, "NULL argument");
    const Plan& P = plan_of(plan);
    if ((sizeof(float2) << P.n) > state_bytes) return fail(QT_EOOM, "state buffer smaller than 2^n amplitudes");
    for (const PlanOp& op : P.ops)
        if (op.kind != 0) return fail(QT_EINVAL, "qt_apply_plan: the plan must hold gates/matrices only");
    ObsGroups og;
    og.final_pass = false;
    return run_single(ctx, plan, reinterpret_cast<float2*>(state_dev), og, {}, 0, 0, 0, 0, nullptr, nullptr, 1,
                      nullptr, false);
}

qt_status qt_reduce_rho(qt_ctx ctx, const void* state_dev, int n, int nq, const int* qubits, double* out) {
    if (!ctx || !state_dev || !qubits || !out) return fail(QT_EINVAL, "NULL argument");
    if (nq < 1 || nq > 6) return fail(QT_EARITY, "qt_reduce_rho: 1..6 qubits");
    uint64_t qmask = 0;
    for (int i = 0; i < nq; ++i) {
        if (qubits[i] < 0 || qubits[i] >= n) return fail(QT_EQUBIT, "qubit out of range");
        qmask |= 1ull << qubits[i];
    }
    if (__builtin_popcountll(qmask) != nq) return fail(QT_EQUBIT, "duplicate qubit");
    QT_CK(cudaSetDevice(ctx->device));
    BatchBufs& B = ctx->bb[0];
    if (finish_batch(B, Plan(), 0, 0, CallOut{}) != QT_OK) return QT_ECUDA;
    const size_t stride = std::max<size_t>(32, (size_t)2 << (2 * nq));
    QT_CK(B.rho_part.ensure(sizeof(double) * (296 * stride + stride)));
    double* partial = B.rho_part.as<double>();
    double* dout = partial + 296 * stride;
    QT_CK(launch_rho_reduce(reinterpret_cast<const float2*>(state_dev), n, qmask, nq, partial, dout, ctx->stream));
    QT_CK(cudaMemcpyAsync(out, dout, sizeof(double) * (2 << (2 * nq)), cudaMemcpyDeviceToHost, ctx->stream));
    QT_CK(cudaStreamSynchronize(ctx->stream));
    return QT_OK;
}

qt_status qt_sample_local(qt_ctx ctx, const void* state_dev, int n_local, int n_total, uint64_t seed, uint64_t traj,
                          int nshots, const int32_t* shot_ids, uint64_t* out) {
    if (!ctx || !state_dev || (nshots > 0 && (!shot_ids || !out)) || nshots < 0 || n_total < n_local)
        return fail(QT_EINVAL, "bad argument");
    if (nshots == 0) return QT_OK;
    qt_plan p = nullptr;
    qt_status e = read_only_plan(n_local, &p);
    if (e != QT_OK) return e;
    ObsGroups og;
    og.ranges.push_back({0, 0});
    og.masks.push_back(0);
    SingleExtras ex;
    ex.n_rng = n_total;
    ex.shot_ids = shot_ids;
    e = run_single(ctx, p, const_cast<float2*>(reinterpret_cast<const float2*>(state_dev)), og, {}, 0, nshots, seed,
                   traj, out, nullptr, 1, nullptr, false, &ex);
    qt_plan_destroy(p);
    return e;
}

qt_status qt_expectation_partials(qt_ctx ctx, const void* state_dev, int n, int n_obs, const qt_pauli* obs,
                                  double* out, double* out_norm) {
    if (!ctx || !state_dev || !out_norm || (n_obs > 0 && (!obs || !out))) return fail(QT_EINVAL, "bad argument");
    qt_plan p = nullptr;
    qt_status e = read_only_plan(n, &p);
    if (e != QT_OK) return e;
    const Plan& P = plan_of(p);
    std::vector<ObsDesc> table;
    ObsGroups og;
    SingleExtras ex;
    ex.out_norm = out_norm;
    if ((e = parse_obs(n, P.T, P.CL, n_obs, obs, table, og)) == QT_OK)
        e = run_single(ctx, p, const_cast<float2*>(reinterpret_cast<const float2*>(state_dev)), og, table, n_obs, 0,
                       0, 0, nullptr, out, 1, nullptr, false, &ex);
    qt_plan_destroy(p);
    return e;
}

}  // extern "C"

// ---------------------------------------------------------------------------
// Diagnostics (not in the header): shared-memory wavefronts per warp store /
// load instruction that the planner's tensor-core layouts imply for trajectory
// `traj` (half-warp model of 8-byte accesses: 16 lanes, 16 bank pairs).
// out[0] = chained readout store instructions (per warp), out[1] = their
// wavefronts, out[2] = run-start fp32 gather loads, out[3] = their wavefronts,
// out[4] = run-end fp32 stores, out[5] = their wavefronts, out[6] = chained
// transitions, out[7] = those whose next gate uses another group bit (no
// two-group overlap).  `out` holds 8 doubles.
// ---------------------------------------------------------------------------
namespace {
uint32_t swz_h(uint32_t L) { return L ^ (((L >> 4) ^ (L >> 8)) & 15u); }
int halfwarp_wavefronts(const uint32_t* addr32) {
    int w = 0;
    for (int h = 0; h < 2; ++h) {
        int cnt[16] = {0};
        int mx = 0;
        for (int l = 0; l < 16; ++l) mx = std::max(mx, ++cnt[(addr32[16 * h + l] >> 3) & 15u]);
        w += mx;
    }
    return w;
}
}  // namespace

extern "C" qt_status qt_plan_bank_stats(qt_plan plan, uint64_t seed, uint64_t traj, double* out) {
    if (!plan || !out) return fail(QT_EINVAL, "NULL argument");
    const Plan& P = plan_of(plan);
    ObsGroups og;
    og.ranges.push_back({0, 0});
    og.masks.push_back(0);
    TrajProgram pg;
    qt_status e = plan_trajectory(P, seed, traj, og, pg);
    if (e != QT_OK) return e;
    for (int i = 0; i < 8; ++i) out[i] = 0;
    const int T = P.T;
    auto fp32_addrs = [&](const GateDesc& G, int warp, int g, int c, uint32_t* a) {
        for (int l = 0; l < 32; ++l) {
            const uint32_t tid = (uint32_t)(warp * 32 + l);
            uint32_t tb = 0;
            for (int i = 0; i < T - 5; ++i) tb |= ((tid >> i) & 1u) << ((G.tpos >> (4 * i)) & 15u);
            uint32_t L = tb;
            for (int m = 0; m < 4; ++m)
                if ((c >> m) & 1) L ^= 1u << ((G.rpos >> (4 * m)) & 15u);
            if (g) L ^= 1u << ((G.rpos >> 16) & 15u);
            a[l] = swz_h(L) << 3;
        }
    };
    for (const PassDesc& ps : pg.passes) {
        for (int gi = 0; gi < ps.gate_count; ++gi) {
            const GateDesc& G = pg.gates[ps.gate_begin + gi];
            if (!(G.k & kGateF16)) continue;
            const bool start = (G.k & kGateRunStart) != 0 || gi == 0 || !(pg.gates[ps.gate_begin + gi - 1].k & kGateF16);
            const bool chained = gi + 1 < ps.gate_count &&
                                 (pg.gates[ps.gate_begin + gi + 1].k & (kGateF16 | kGateRunStart)) == kGateF16;
            if (chained) {
                out[6] += 1;
                out[7] += G.xu[4] != (uint16_t)16384;  // tc::kF16GroupBytes
            }
            uint32_t a[32];
            for (int warp = 0; warp < 4; ++warp)
                for (int g = 0; g < 2; ++g)
                    for (int c = 0; c < 16; ++c) {
                        if (start) {
                            fp32_addrs(G, warp, g, c, a);
                            out[2] += 1;
                            out[3] += halfwarp_wavefronts(a);
                        }
                        if (chained) {
                            if (G.pair && (c & 1)) continue;  // stored with c - 1 (16-byte store)
                            for (int l = 0; l < 32; ++l) {
                                const uint32_t tid = (uint32_t)(warp * 32 + l);
                                uint32_t o = 0;
                                for (int i = 0; i < 7; ++i)
                                    if ((tid >> i) & 1u) o ^= G.xu[5 + i];
                                for (int m = 0; m < 4; ++m)
                                    if ((c >> m) & 1) o ^= G.xu[m];
                                a[l] = o;
                            }
                            out[0] += 1;
                            if (G.pair) {  // quarter-warps of 8 lanes x 16 bytes, 8 chunks per 128 bytes
                                for (int qw = 0; qw < 4; ++qw) {
                                    int cnt[8] = {0}, mx = 0;
                                    for (int l = 0; l < 8; ++l) mx = std::max(mx, ++cnt[(a[8 * qw + l] >> 4) & 7u]);
                                    out[1] += mx;
                                }
                            } else {
                                out[1] += halfwarp_wavefronts(a);
                            }
                        } else {
                            fp32_addrs(G, warp, g, c, a);
                            out[4] += 1;
                            out[5] += halfwarp_wavefronts(a);
                        }
                    }
        }
    }
    return QT_OK;
}

// Diagnostic (undeclared, like qt_plan_bank_stats): the pass / fused-gate structure of
// one trajectory's program.  out = [n_pass, then per pass: tile_mask, flags,
// gate_count, then per gate: global qubit mask of its (padded) matrix bits, k, 5 words of v2 units].
extern "C" qt_status qt_plan_dump(qt_plan plan, uint64_t seed, uint64_t traj, int64_t* out, int64_t cap) {
    if (!plan || !out) return fail(QT_EINVAL, "NULL argument");
    const Plan& P = plan_of(plan);
    ObsGroups og;
    og.ranges.push_back({0, 0});
    og.masks.push_back(0);
    TrajProgram pg;
    qt_status e = plan_trajectory(P, seed, traj, og, pg);
    if (e != QT_OK) return e;
    int64_t w = 0;
    auto put = [&](int64_t v) {
        if (w < cap) out[w] = v;
        ++w;
    };
    put((int64_t)pg.passes.size());
    for (const PassDesc& ps : pg.passes) {
        put((int64_t)ps.tile_mask);
        put(ps.flags);
        put(ps.gate_count);
        for (int g = 0; g < ps.gate_count; ++g) {
            const GateDesc& G = pg.gates[ps.gate_begin + g];
            const int k = (G.k & kGateTC) ? 4 : (G.k & 0xff);
            uint64_t m = 0;
            if (G.k & kGateV2) {  // v2 units: fp32 byte offset of a tile bit b has its top bit at b + 3
                for (int j = 0; j < 4; ++j) m |= 1ull << ps.tq[31 - __builtin_clz((uint32_t)v2_units(G)[j]) - 3];
            } else {
                for (int j = 0; j < k; ++j) m |= 1ull << ps.tq[(G.rpos >> (4 * j)) & 15u];
            }
            put((int64_t)m);
            put(G.k);
            // v2 layout units (20 x uint16, desc.hpp v2_units), zeros for other kernels
            uint16_t u[20] = {0};
            if (G.k & kGateV2) std::memcpy(u, v2_units(G), sizeof u);
            for (int j = 0; j < 5; ++j) {
                int64_t x = 0;
                std::memcpy(&x, u + 4 * j, 8);
                put(x);
            }
        }
    }
    return w <= cap ? QT_OK : fail(QT_EINVAL, "plan dump: capacity too small");
}
