// oracle/tools/psf_driver.cpp — TEST INFRASTRUCTURE ONLY.
//
// Runs the UNMODIFIED reference library (oracle/_ref/libwaveblur_ref.so) on the PSF side of
// the path (operators.cpp): generate_psf for every PsfSpec kind, convolve / apply_adjoint of
// the synthetic scene, and degrade. Writes raw little-endian f64 binaries into DIR for
// oracle/make_psf_golden.py (tests/golden/psf_cases.npz).
//
//   psf_driver DIR
#include <cstdio>
#include <fstream>
#include <string>
#include <vector>

#include "waveblur/image.hpp"
#include "waveblur/operators.hpp"

using namespace waveblur;

namespace {

void write_bin(const std::string& path, const std::vector<double>& v) {
    std::ofstream f(path, std::ios::binary);
    f.write(reinterpret_cast<const char*>(v.data()), static_cast<std::streamsize>(v.size() * sizeof(double)));
}

struct Case {
    std::string name;
    PsfSpec spec;
    std::vector<std::size_t> dims;
};

}  // namespace

int main(int argc, char** argv) {
    if (argc < 2) return 2;
    const std::string dir = argv[1];
    const std::vector<Case> cases = {
        {"gauss3_64", GaussianSpec{3.0}, {64, 64}},
        {"gauss_delta_32", GaussianSpec{0.5}, {32}},
        {"skewed5_64", SkewedGaussianSpec{5.0}, {64, 64}},
        {"skewed3_128_1d", SkewedGaussianSpec{3.0}, {128}},
        {"motion_42_64", MotionSpec{5, 8.0, 1.0, 42}, {64, 64}},
        {"motion_7_32", MotionSpec{5, 8.0, 1.0, 7}, {32, 32}},
        {"motion_default_256", MotionSpec{}, {256, 256}},
        {"motion_3_128_1d", MotionSpec{4, 6.0, 1.5, 3}, {128}},
        {"airy4_64", AirySpec{4.0}, {64, 64}},
        {"airy2_128_1d", AirySpec{2.0}, {128}},
        {"defocus6_64", DefocusSpec{6.0}, {64, 64}},
        {"defocus3_128_1d", DefocusSpec{3.0}, {128}},
        {"skewed8_1024", SkewedGaussianSpec{8.0}, {1024, 1024}},
    };
    std::FILE* idx = std::fopen((dir + "/index.txt").c_str(), "w");
    for (const auto& c : cases) {
        Psf p = generate_psf(c.spec, c.dims);
        write_bin(dir + "/" + c.name + ".bin", p.kernel.v);
        std::fprintf(idx, "%s %s", c.name.c_str(), psf_spec_string(c.spec).c_str());
        for (auto d : c.dims) std::fprintf(idx, " %zu", d);
        std::fprintf(idx, "\n");
    }
    std::fclose(idx);
    // convolution, its adjoint and degrade on the synthetic scene with the motion kernel
    const std::vector<std::size_t> dims = {64, 64};
    Psf p = generate_psf(MotionSpec{5, 8.0, 1.0, 42}, dims);
    Image u = synthetic_scene(dims);
    write_bin(dir + "/scene64.bin", u.v);
    write_bin(dir + "/conv64.bin", convolve(u, p).v);
    write_bin(dir + "/adj64.bin", apply_adjoint(u, p).v);
    write_bin(dir + "/degrade64.bin", degrade(u, DegradationModel{p, 1e-2, 11}).v);
    write_bin(dir + "/noise64.bin", add_noise(u, 1e-2, 11).v);
    return 0;
}
