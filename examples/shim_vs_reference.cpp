// Integration example: a reference caller switches from ofdmradar:: to ofdmradar::b200::
// (include/ofdmradar_b200.hpp) and gets the same receiver outputs.  Links the reference's
// own receiver sources (oracle/_ref/libofdmref.so) next to the B200 library and compares
// them on seeded grids: spectral_division, dft_ce, periodogram (Hamming + padding),
// extract_peaks on the same map, and sft_iterate.  Exit code 0 = all within the parity
// bars (maps <= 1e-4 of the peak, bins / SFT supports identical).
#include <cmath>
#include <cstdio>
#include <set>
#include <vector>

#include "ofdmradar/estimation.hpp"
#include "ofdmradar/periodogram.hpp"
#include "ofdmradar/rng.hpp"
#include "ofdmradar/sft.hpp"
#include "ofdmradar_b200.hpp"

using namespace ofdmradar;

static ComplexGrid grid(std::size_t n, std::size_t m, std::uint64_t seed, double tone_amp) {
    ComplexGrid g(n, m, AxisTag::SubcarrierSymbol);
    Rng rng(seed);
    const double tp = 6.283185307179586476925286766559;
    for (std::size_t k = 0; k < n; ++k)
        for (std::size_t l = 0; l < m; ++l) {
            const double a = rng.normal(), b = rng.normal();
            g.at(k, l) = cplx(a, b) * std::sqrt(0.5) +
                         tone_amp * std::polar(1.0, tp * (-double(k) * 37.0 / n + double(l) * 11.0 / m));
        }
    return g;
}

static double rel_max_diff(const RealGrid& a, const RealGrid& b) {
    double d = 0.0, pk = 0.0;
    for (std::size_t i = 0; i < a.size(); ++i) {
        d = std::max(d, std::abs(a.storage()[i] - b.storage()[i]));
        pk = std::max(pk, a.storage()[i]);
    }
    return d / pk;
}

int main() {
    int fails = 0;
    // periodogram, Hamming, zero padding
    const ComplexGrid h = grid(256, 64, 7, 3.0);
    const Window2d w = make_window(WindowKind::Hamming, 256, 64);
    const RealGrid pr = periodogram(h, w, 512, 128);
    const RealGrid pg = b200::periodogram(h, w, 512, 128);
    const double e1 = rel_max_diff(pr, pg);
    std::printf("periodogram 256x64 -> 512x128 hamming: max |dP|/max P = %.3e\n", e1);
    fails += e1 > 1e-4;
    // extract_peaks on the reference map
    WaveformConfig wc;
    wc.n_subcarriers = 256;
    wc.n_symbols = 64;
    wc.n_prime = 512;
    wc.m_prime = 128;
    const double eta = detection_threshold(1.0, 1e-2, w.power_factor());
    const auto mask = threshold_mask(pr, eta);
    const auto dr = extract_peaks(pr, mask, 8, wc);
    const auto dg = b200::extract_peaks(pr, mask, 8, wc);
    bool same = dr.size() == dg.size();
    for (std::size_t i = 0; same && i < dr.size(); ++i)
        same = dr[i].delay_bin == dg[i].delay_bin && dr[i].doppler_bin == dg[i].doppler_bin &&
               dr[i].range_m == dg[i].range_m && dr[i].velocity_mps == dg[i].velocity_mps;
    std::printf("extract_peaks: %zu reference detections, identical = %d\n", dr.size(), int(same));
    fails += !same;
    // dft_ce
    const ComplexGrid c1 = dft_ce(h, 32), c2 = b200::dft_ce(h, 32);
    double dm = 0.0, am = 0.0;
    for (std::size_t i = 0; i < c1.size(); ++i) {
        dm = std::max(dm, std::abs(c1.storage()[i] - c2.storage()[i]));
        am = std::max(am, std::abs(c1.storage()[i]));
    }
    std::printf("dft_ce L=32: max |dH|/max |H| = %.3e\n", dm / am);
    fails += dm / am > 1e-5;
    // spectral_division + ConfigError on a zero cell
    ComplexGrid x = grid(256, 64, 9, 0.0);
    const ComplexGrid q1 = spectral_division(h, x), q2 = b200::spectral_division(h, x);
    double qm = 0.0, qa = 0.0;
    for (std::size_t i = 0; i < q1.size(); ++i) {
        qm = std::max(qm, std::abs(q1.storage()[i] - q2.storage()[i]));
        qa = std::max(qa, std::abs(q1.storage()[i]));
    }
    std::printf("spectral_division: max rel %.3e\n", qm / qa);
    fails += qm / qa > 1e-5;
    x.at(3, 4) = cplx(0, 0);
    bool threw = false;
    try {
        b200::spectral_division(h, x);
    } catch (const ConfigError&) {
        threw = true;
    }
    std::printf("zero X cell -> ConfigError: %d\n", int(threw));
    fails += !threw;
    // FPS-SFT on a 5-sparse 64 x 32 grid
    ComplexGrid s(64, 32, AxisTag::SubcarrierSymbol);
    const int ks[5] = {3, 17, 29, 40, 55}, ls[5] = {1, 9, 14, 22, 30};
    for (std::size_t a = 0; a < 64; ++a)
        for (std::size_t b = 0; b < 32; ++b) {
            cplx acc(0, 0);
            for (int t = 0; t < 5; ++t)
                acc += (0.6 + 0.3 * t) * std::polar(1.0, 6.283185307179586 * (double(a) * ks[t] / 64.0 +
                                                                           double(b) * ls[t] / 32.0 + 0.1 * t));
            s.at(a, b) = acc;
        }
    SftConfig sc;
    sc.seed = 11;
    const auto s1 = sft_iterate(s, sc), s2 = b200::sft_iterate(s, sc);
    std::set<std::pair<long, long>> a1, a2;
    for (const auto& e : s1.entries) a1.insert({e.k, e.l});
    for (const auto& e : s2.entries) a2.insert({e.k, e.l});
    std::printf("sft_iterate: reference %zu entries, b200 %zu entries, same support = %d, iterations %zu/%zu\n",
                s1.entries.size(), s2.entries.size(), int(a1 == a2), s1.iterations, s2.iterations);
    fails += a1 != a2;
    // detections_from_spectrum / sft_detect (sft.hpp:67-75) on the same spectrum and grid
    {
        const auto d1 = detections_from_spectrum(s1, 64, 32, wc, 0.01, 1e-2, 4);
        const auto d2 = b200::detections_from_spectrum(s1, 64, 32, wc, 0.01, 1e-2, 4);
        bool same = d1.size() == d2.size();
        for (std::size_t i = 0; same && i < d1.size(); ++i)
            same = d1[i].delay_bin == d2[i].delay_bin && d1[i].doppler_bin == d2[i].doppler_bin &&
                   d1[i].peak_power == d2[i].peak_power && d1[i].range_m == d2[i].range_m &&
                   d1[i].velocity_mps == d2[i].velocity_mps;
        SftConfig sd;
        sd.seed = 11;
        const auto t1 = sft_detect(s, wc, sd, 0.01, 1e-2, 5), t2 = b200::sft_detect(s, wc, sd, 0.01, 1e-2, 5);
        bool same2 = t1.size() == t2.size();
        for (std::size_t i = 0; same2 && i < t1.size(); ++i)
            same2 = t1[i].delay_bin == t2[i].delay_bin && t1[i].doppler_bin == t2[i].doppler_bin;
        std::printf("detections_from_spectrum: %zu/%zu identical = %d; sft_detect %zu/%zu identical bins = %d\n",
                    d1.size(), d2.size(), int(same), t1.size(), t2.size(), int(same2));
        fails += !same || !same2;
    }
    // estimate_noise_power on the reference's own periodogram
    {
        const double pfw = w.power_factor();
        const double e1 = estimate_noise_power(pr, pfw), e2 = b200::estimate_noise_power(pr, pfw);
        const bool ok = std::abs(e1 - e2) <= 1e-6 * e1;
        std::printf("estimate_noise_power: reference %.9g, b200 %.9g, ok = %d\n", e1, e2, int(ok));
        fails += !ok;
    }
    // OFDM front end: b200 modulate -> reference demodulate, reference modulate -> b200 demodulate
    {
        WaveformConfig ow = wc;
        ow.n_subcarriers = 256;
        ow.n_symbols = 16;
        ow.n_cp = 32;
        ComplexGrid xg(256, 16, AxisTag::SubcarrierSymbol);
        for (std::size_t a = 0; a < 256; ++a)
            for (std::size_t b = 0; b < 16; ++b) xg.at(a, b) = std::polar(1.0, 0.7 * double(a * 16 + b));
        const auto st_ref = ofdm_modulate(xg, ow), st_b200 = b200::ofdm_modulate(xg, ow);
        double e_mod = 0, peak = 0;
        for (std::size_t i = 0; i < st_ref.size(); ++i) {
            e_mod = std::max(e_mod, std::abs(st_ref[i] - st_b200[i]));
            peak = std::max(peak, std::abs(st_ref[i]));
        }
        const ComplexGrid d_ref = ofdm_demodulate(st_ref, ow), d_b200 = b200::ofdm_demodulate(st_ref, ow);
        double e_dem = 0;
        for (std::size_t a = 0; a < 256; ++a)
            for (std::size_t b = 0; b < 16; ++b) e_dem = std::max(e_dem, std::abs(d_ref.at(a, b) - d_b200.at(a, b)));
        const bool ok = e_mod <= 1e-5 * peak && e_dem <= 1e-5;
        std::printf("ofdm_modulate/demodulate: max err %.3g / %.3g, ok = %d\n", e_mod / peak, e_dem, int(ok));
        fails += !ok;
    }
    std::printf("%s\n", fails ? "FAIL" : "OK");
    return fails ? 1 : 0;
}
