// C-ABI over the kFkB stage executor (include/ptk.h ptk_exec_*).
#include <cstring>
#include <exception>
#include <string>

#include "../../../include/ptk.h"
#include "../host/json_out.h"
#include "errors.h"
#include "executor.h"
#include "pipetune/errors.hpp"

#include "capi_handles.h"

struct ptk_exec {
    ptk::Executor impl;
    ptk_stage stage_view;
    explicit ptk_exec(const ptk_exec_config& c) : impl(c), stage_view(&impl.stage(), false) {}
};

namespace {

template <class F>
int guarded(const char* what, F&& f) {
    try {
        f();
        return PTK_OK;
    } catch (const pipetune::ConfigError& e) {
        return ptk::set_error(PTK_ERR_ARG, std::string(what) + ": " + e.what());
    } catch (const pipetune::PlanError& e) {
        return ptk::set_error(PTK_ERR_PLAN, std::string(what) + ": " + e.what());
    } catch (const pipetune::DeadlockDetected& e) {
        return ptk::set_error(PTK_ERR_DEADLOCK, std::string(what) + ": " + e.what());
    } catch (const pipetune::InfeasibleModel& e) {
        return ptk::set_error(PTK_ERR_INFEASIBLE, std::string(what) + ": " + e.what());
    } catch (const std::logic_error& e) {  // invalid_argument, out-of-order calls
        return ptk::set_error(PTK_ERR_ARG, std::string(what) + ": " + e.what());
    } catch (const std::exception& e) {
        return ptk::set_error(PTK_ERR_CUDA, std::string(what) + ": " + e.what());
    }
}

float ms_between(cudaEvent_t a, cudaEvent_t b) {
    float ms = 0.f;
    cudaEventElapsedTime(&ms, a, b);
    return ms;
}

}  // namespace

#define EX_CHECK(ex) \
    if (!(ex)) return ptk::set_error(PTK_ERR_ARG, "null executor")

extern "C" int ptk_exec_create(const ptk_exec_config* cfg, ptk_exec** out) {
    if (!cfg || !out) return ptk::set_error(PTK_ERR_ARG, "ptk_exec_create: null argument");
    return guarded("ptk_exec_create", [&] { *out = new ptk_exec(*cfg); });
}

extern "C" int ptk_exec_destroy(ptk_exec* ex) {
    delete ex;
    return PTK_OK;
}

extern "C" int ptk_exec_export(ptk_exec* ex, void* buf, size_t cap, size_t* written) {
    EX_CHECK(ex);
    return guarded("ptk_exec_export", [&] {
        const auto h = ex->impl.export_handles();
        if (written) *written = h.size();
        if (!buf || cap < h.size()) throw std::invalid_argument("buffer too small");
        std::memcpy(buf, h.data(), h.size());
    });
}

extern "C" int ptk_exec_import(ptk_exec* ex, int peer, const void* buf, size_t n) {
    EX_CHECK(ex);
    return guarded("ptk_exec_import",
                   [&] { ex->impl.import_peer(peer, static_cast<const uint8_t*>(buf), n); });
}

extern "C" int ptk_exec_connect_local(ptk_exec* ex, int peer, ptk_exec* other) {
    EX_CHECK(ex);
    if (!other) return ptk::set_error(PTK_ERR_ARG, "null peer");
    return guarded("ptk_exec_connect_local", [&] { ex->impl.connect_local(peer, other->impl); });
}

extern "C" int ptk_exec_set_plan(ptk_exec* ex, int k, int b) {
    EX_CHECK(ex);
    return guarded("ptk_exec_set_plan", [&] { ex->impl.set_plan(k, b); });
}

extern "C" int ptk_exec_set_plan_groups(ptk_exec* ex, int b, const int* sizes, int n) {
    EX_CHECK(ex);
    if (n < 1 || sizes == nullptr) return ptk::set_error(PTK_ERR_ARG, "ptk_exec_set_plan_groups: empty group list");
    return guarded("ptk_exec_set_plan_groups",
                   [&] { ex->impl.set_plan_groups(b, std::vector<int>(sizes, sizes + n)); });
}

extern "C" int ptk_exec_set_trace(ptk_exec* ex, int link, double base, int64_t latency, int nseg, const int64_t* s,
                                  const int64_t* e, const double* a) {
    EX_CHECK(ex);
    return guarded("ptk_exec_set_trace", [&] {
        ptk::EmuTrace t;
        t.active = base > 0.0;
        t.base_bytes_per_ns = base;
        t.latency_ns = latency;
        for (int i = 0; i < nseg; ++i) t.segments.push_back({s[i], e[i], a[i]});
        ex->impl.set_trace(link, t);
    });
}

extern "C" int ptk_exec_set_epoch(ptk_exec* ex, int64_t epoch) {
    EX_CHECK(ex);
    return guarded("ptk_exec_set_epoch", [&] { ex->impl.set_epoch(epoch); });
}

extern "C" int ptk_exec_set_contender(ptk_exec* ex, int on) {
    EX_CHECK(ex);
    return guarded("ptk_exec_set_contender", [&] { ex->impl.set_contender(on != 0); });
}

extern "C" int64_t ptk_globaltimer(void) {
    try {
        return ptk::device_globaltimer(0);
    } catch (...) {
        return -1;
    }
}

extern "C" int ptk_exec_run_iteration(ptk_exec* ex, int iter, const int32_t* host_tokens) {
    EX_CHECK(ex);
    return guarded("ptk_exec_run_iteration", [&] { ex->impl.run_iteration(iter, host_tokens); });
}

extern "C" int ptk_exec_begin_iteration(ptk_exec* ex, int iter, const int32_t* host_tokens) {
    EX_CHECK(ex);
    return guarded("ptk_exec_begin_iteration", [&] { ex->impl.begin_iteration(iter, host_tokens); });
}

extern "C" int ptk_exec_enqueue_next(ptk_exec* ex, int* more) {
    EX_CHECK(ex);
    return guarded("ptk_exec_enqueue_next", [&] {
        const bool m = ex->impl.enqueue_next();
        if (more) *more = m ? 1 : 0;
    });
}

extern "C" int ptk_exec_run_local(ptk_exec* const* stages, int n, int iter, const int32_t* host_tokens) {
    if (stages == nullptr || n < 1) return ptk::set_error(PTK_ERR_ARG, "ptk_exec_run_local: empty stage list");
    return guarded("ptk_exec_run_local", [&] {
        std::vector<ptk::Executor*> v;
        for (int i = 0; i < n; ++i) {
            if (stages[i] == nullptr) throw std::invalid_argument("null stage");
            v.push_back(&stages[i]->impl);
        }
        ptk::run_local_pipeline(v, iter, host_tokens);
    });
}

extern "C" int ptk_exec_set_deadlock_timeout(ptk_exec* ex, double seconds) {
    EX_CHECK(ex);
    if (!(seconds > 0.0)) return ptk::set_error(PTK_ERR_ARG, "ptk_exec_set_deadlock_timeout: seconds must be > 0");
    ex->impl.set_deadlock_timeout(seconds);
    return PTK_OK;
}

extern "C" int ptk_exec_set_send_streams(ptk_exec* ex, int per_link) {
    EX_CHECK(ex);
    ex->impl.set_send_streams_per_link(per_link != 0);
    return PTK_OK;
}

extern "C" int ptk_exec_finish_iteration(ptk_exec* ex, double* ms) {
    EX_CHECK(ex);
    return guarded("ptk_exec_finish_iteration", [&] {
        const double v = ex->impl.finish_iteration();
        if (ms) *ms = v;
    });
}

extern "C" int ptk_exec_read_loss(ptk_exec* ex, float* loss) {
    EX_CHECK(ex);
    return guarded("ptk_exec_read_loss", [&] { *loss = ex->impl.read_loss(); });
}

extern "C" int ptk_exec_timeline_json(ptk_exec* ex, char* buf, size_t cap, size_t* written) {
    EX_CHECK(ex);
    return guarded("ptk_exec_timeline_json", [&] {
        pipetune::json::Writer w;
        cudaEvent_t t0 = ex->impl.iteration_start();
        auto ns = [&](cudaEvent_t e) { return static_cast<long long>(ms_between(t0, e) * 1e6 + 0.5); };
        w.begin_obj().key("compute").begin_arr();
        for (const auto& r : ex->impl.comp_records())
            w.begin_arr().v(r.node).v(r.kind).v(r.mb).v(ns(r.start)).v(ns(r.end)).end_arr();
        w.end_arr().key("xfer").begin_arr();
        for (const auto& r : ex->impl.xfer_records())
            w.begin_arr().v(r.link).v(r.mb).v(r.bytes).v(ns(r.start)).v(ns(r.end)).end_arr();
        w.end_arr();
        w.key("launches").num(ex->impl.kernel_launches());
        w.key("h2d_bytes").num(ex->impl.h2d_bytes());
        w.key("k").num(ex->impl.plan_k());
        w.key("b").num(ex->impl.plan_b());
        w.key("groups").begin_arr();
        for (int n : ex->impl.plan_groups()) w.v(n);
        w.end_arr();
        w.key("t0_globaltimer").num(ex->impl.iteration_start_globaltimer());
        w.key("stage").num(ex->impl.cfg().stage);
        w.end_obj();
        if (written) *written = w.out.size() + 1;
        if (!buf || cap < w.out.size() + 1) throw std::invalid_argument("buffer too small");
        std::memcpy(buf, w.out.c_str(), w.out.size() + 1);
    });
}

extern "C" int ptk_exec_probe_link(ptk_exec* ex, int link, int64_t bytes, int repeats, int64_t* out_ns) {
    EX_CHECK(ex);
    return guarded("ptk_exec_probe_link", [&] {
        const auto v = ex->impl.probe_link(link, bytes, repeats);
        for (size_t i = 0; i < v.size(); ++i) out_ns[i] = v[i];
    });
}

extern "C" int ptk_exec_profile_compute(ptk_exec* ex, int b, int repeats, int64_t* f, int64_t* bw) {
    EX_CHECK(ex);
    return guarded("ptk_exec_profile_compute", [&] { ex->impl.profile_compute(b, repeats, f, bw); });
}

extern "C" int ptk_exec_gemm_timing(ptk_exec* ex, int enable, double* total_flops, double* total_ms,
                                    long* launches) {
    EX_CHECK(ex);
    return guarded("ptk_exec_gemm_timing", [&] {
        ptk::GemmTiming& t = ex->impl.stage().gemm_timing();
        ex->impl.stage().collect_timing();
        if (total_flops) *total_flops = t.total_flops;
        if (total_ms) *total_ms = t.total_ms;
        if (launches) *launches = t.launches;
        if (enable >= 0) {
            t.armed = enable != 0;
            t.enabled = t.armed;
            if (t.armed) t.stride = enable > 1 ? enable : 8;  // executor: time one micro-batch in `stride`
            t.total_flops = t.total_ms = 0.0;
            t.launches = 0;
        }
    });
}

extern "C" ptk_stage* ptk_exec_stage(ptk_exec* ex) { return ex ? &ex->stage_view : nullptr; }

extern "C" int ptk_exec_set_wgrad_pairs(ptk_exec* ex, int on) {
    if (ex == nullptr) return ptk::set_error(PTK_ERR_ARG, "ptk_exec_set_wgrad_pairs: null executor");
    return guarded("ptk_exec_set_wgrad_pairs", [&] { ex->impl.stage().set_wgrad_pairs(on != 0); });
}

extern "C" int ptk_exec_set_defer_optimizer(ptk_exec* ex, int defer) {
    EX_CHECK(ex);
    return guarded("ptk_exec_set_defer_optimizer", [&] { ex->impl.set_defer_optimizer(defer != 0); });
}

extern "C" int ptk_exec_compute_stream(ptk_exec* ex, void** stream) {
    EX_CHECK(ex);
    if (stream == nullptr) return ptk::set_error(PTK_ERR_ARG, "ptk_exec_compute_stream: null output");
    *stream = static_cast<void*>(ex->impl.compute_stream());
    return PTK_OK;
}
