// histogram.cu -- weight_histogram (observables.hpp:114-176) orchestration; kernels and rationale: histogram.cuh.
#include "engine.cuh"
#include "histogram.cuh"

namespace pb {

void Engine::weight_histogram(const double2* cvec, uint32_t n, uint64_t bins, pb200_weight_hist* out, uint64_t* rank,
                              double* weight, uint64_t cap, uint64_t* npts_out) {
    Ctl* c = dctl();
    weights.ensure(size_t(n) * 8 + 8);
    sort_out.ensure(size_t(n) * 8 + 8);
    sort_tmp.ensure(size_t(n) * 8 + 8);
    PB_CUDA(cudaMemsetAsync(&c->select, 0, sizeof(SelectCtl), stream));
    weights_kernel<<<grid_for(n), NT, 0, stream>>>(cvec, n, weights.as<double>(), partials.as<double>(), &c->select);
    check_launch();

    // ---- stable LSD radix sort of ~bits(w), 8 bits per pass: count -> scan -> scatter
    unsigned long long* ka = sort_out.as<unsigned long long>();
    unsigned long long* kb = sort_tmp.as<unsigned long long>();
    rs_make_keys_kernel<<<grid_for(n), NT, 0, stream>>>(weights.as<double>(), n, ka);
    check_launch();
    const uint32_t ntiles = (n + RS_TILE - 1) / RS_TILE;
    const uint64_t ncounts = uint64_t(ntiles) * RS_BINS;
    hist_counts.ensure((ncounts + 1) * 4);
    for (int shift = 0; shift < 64; shift += RS_BITS) {
        rs_count_kernel<<<ntiles, NT, 0, stream>>>(ka, n, shift, ntiles, hist_counts.as<uint32_t>());
        check_launch();
        exclusive_scan(hist_counts.as<uint32_t>(), ncounts);
        rs_scatter_kernel<<<ntiles, NT, 0, stream>>>(ka, n, shift, ntiles, hist_counts.as<uint32_t>(), kb);
        check_launch();
        std::swap(ka, kb);
    }
    // 8 passes: the sorted keys are back in sort_out (ka)

    const SelectCtl sc = read_back<SelectCtl>(&c->select);
    const uint64_t m = sc.support;  // weights are >= 0: the positive ones lead the descending order
    if (m == 0) throw PacesError("weight histogram: empty state");

    // ---- marks + tail slope over the m leading (positive) weights
    const uint32_t mtiles = uint32_t((m + RS_TILE - 1) / RS_TILE);
    hist_tiles.ensure(size_t(mtiles) * 8 + 8);
    hist_res.ensure(sizeof(WeightHistDev));
    WeightHistDev* res = hist_res.as<WeightHistDev>();
    PB_CUDA(cudaMemsetAsync(res, 0, sizeof(WeightHistDev), stream));
    wh_tile_sums_kernel<<<mtiles, NT, 0, stream>>>(ka, uint32_t(m), hist_tiles.as<double>());
    check_launch();
    wh_scan_tiles_kernel<<<1, NT, 0, stream>>>(hist_tiles.as<double>(), mtiles, &res->total);
    check_launch();
    const uint32_t lo = uint32_t(m / 10);  // the tail: the last nine deciles (observables.hpp:149)
    const int mgrid = int(std::min<uint64_t>(mtiles, uint64_t(sm_count) * 8));
    wh_marks_slope_kernel<<<mgrid, NT, 0, stream>>>(ka, uint32_t(m), hist_tiles.as<double>(), lo, partials.as<double>(),
                                                    res);
    check_launch();
    const uint64_t npts = (bins == 0 || m <= bins) ? m : bins;
    const uint64_t cnt = std::min<uint64_t>(npts, cap);
    const bool want_curve = cnt > 0 && (rank || weight);
    if (want_curve) {
        hist_curve.ensure(size_t(cnt) * 16 + 16);
        wh_sample_kernel<<<grid_for(cnt), NT, 0, stream>>>(ka, m, npts, cnt, hist_curve.as<unsigned long long>(),
                                                           hist_curve.as<double>() + cnt);
        check_launch();
    }
    const WeightHistDev h = read_back<WeightHistDev>(res);
    if (want_curve) {
        if (rank)
            PB_CUDA(cudaMemcpyAsync(rank, hist_curve.p, size_t(cnt) * 8, cudaMemcpyDeviceToHost, stream));
        if (weight)
            PB_CUDA(cudaMemcpyAsync(weight, hist_curve.as<double>() + cnt, size_t(cnt) * 8, cudaMemcpyDeviceToHost,
                                    stream));
        sync();
    }
    out->support = m;
    uint64_t* marks[4] = {&out->q50, &out->q90, &out->q99, &out->q9999};
    for (int j = 0; j < 4; ++j) *marks[j] = std::min<uint64_t>(h.below[j] + 1, m);
    out->tail_exponent = 0;
    if (m - lo >= 2) {
        const double k = double(m - lo);
        const double denom = k * h.sums[2] - h.sums[0] * h.sums[0];
        out->tail_exponent = denom != 0 ? (k * h.sums[3] - h.sums[0] * h.sums[1]) / denom : 0.0;
    }
    if (npts_out) *npts_out = npts;
}

}  // namespace pb
