// gen_io_golden.cpp — TEST INFRASTRUCTURE ONLY.  Writes the golden files for
// the file-format parity tests (tests/test_io.py) with the reference's own
// writers: save_raw (io_raw.cpp:120-140) for an f32 volume, a u16 label
// volume and a 3-channel field, and save_checkpoint (checkpoint.cpp:85-104)
// for two small model configurations.  Built from the reference sources where
// they lie by oracle/gen_io_golden.sh; the outputs are committed under
// tests/golden/io/ so the tests never need /root/reference.
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <fstream>
#include <string>
#include <vector>

#include "mdreg/engine.hpp"
#include "mdreg/io.hpp"

using namespace mdreg;

// a single-file NIfTI-1 image (the header fields load_nifti reads,
// nifti.cpp:36-60; everything else zero)
static void write_nifti(const std::string &path, int16_t datatype, int16_t bitpix, Dims3 d,
                        const void *data, size_t bytes, float px, float py, float pz,
                        float slope, float inter) {
    char hdr[352] = {};
    const int32_t sizeof_hdr = 348;
    std::memcpy(hdr, &sizeof_hdr, 4);
    const int16_t dim[8] = {3, (int16_t)d.h, (int16_t)d.w, (int16_t)d.l, 1, 1, 1, 1};
    std::memcpy(hdr + 40, dim, sizeof dim);
    std::memcpy(hdr + 70, &datatype, 2);
    std::memcpy(hdr + 72, &bitpix, 2);
    const float pixdim[8] = {1.0f, px, py, pz, 0, 0, 0, 0};
    std::memcpy(hdr + 76, pixdim, sizeof pixdim);
    const float vox_offset = 352.0f;
    std::memcpy(hdr + 108, &vox_offset, 4);
    std::memcpy(hdr + 112, &slope, 4);
    std::memcpy(hdr + 116, &inter, 4);
    std::memcpy(hdr + 344, "n+1", 4);
    std::ofstream f(path, std::ios::binary | std::ios::trunc);
    f.write(hdr, sizeof hdr);
    f.write(static_cast<const char *>(data), (std::streamsize)bytes);
}

int main(int argc, char **argv) {
    const std::string out = argc > 1 ? argv[1] : ".";
    const Dims3 d{5, 4, 3};
    Volume v(d, 0.0f, {1.0f, 0.8f, 1.5f});
    for (std::size_t i = 0; i < v.data.size(); ++i)
        v.data[i] = 0.25f * static_cast<float>(i) - 3.0f + 1e-3f * std::sin(static_cast<float>(i));
    save_raw(v, out + "/vol");
    LabelVolume lab(d, {0.5f, 0.5f, 2.0f});
    for (std::size_t i = 0; i < lab.data.size(); ++i) lab.data[i] = static_cast<int>((i * 7) % 11);
    lab.data[3] = 65535;
    save_raw(lab, out + "/labels");
    DisplacementField f(d);
    for (std::size_t i = 0; i < f.data.size(); ++i)
        f.data[i] = 0.1f * static_cast<float>(i % 13) - 0.6f;
    save_raw(f, out + "/field");

    ModelConfig a = ModelConfig::small_preset();
    a.encoder.base_channels = 1;
    a.heads_per_level = {2, 2, 1, 1, 1};
    a.head_dim = 2;
    auto pa = init_model<float>(a, 3);
    save_checkpoint(out + "/ckpt_a.mdt", pa);
    ModelConfig b = a;
    b.encoder.leaky_slope = 0.1f;
    b.diffeomorphic = true;
    b.ss_steps = 5;
    b.heads_per_level = {3, 2, 2, 1, 1};
    b.head_dim = 1;
    auto pb = init_model<float>(b, 9);
    save_checkpoint(out + "/ckpt_b.mdt", pb);
    // NIfTI: u8, i16 with slope/intercept, f32 unscaled with a non-positive
    // pixdim (spacing falls back to 1); the expected volumes are what the
    // reference's load_nifti returns, stored with save_raw
    const Dims3 nd{6, 5, 4};
    const size_t nn = (size_t)nd.h * nd.w * nd.l;
    std::vector<uint8_t> u8(nn);
    std::vector<int16_t> i16(nn);
    std::vector<float> f32(nn);
    for (size_t i = 0; i < nn; ++i) {
        u8[i] = (uint8_t)((i * 37) % 256);
        i16[i] = (int16_t)((int)((i * 911) % 4001) - 2000);
        f32[i] = 0.37f * (float)i - 20.0f;
    }
    write_nifti(out + "/img_u8.nii", 2, 8, nd, u8.data(), nn, 1.2f, 1.0f, 0.9f, 0.0f, 0.0f);
    write_nifti(out + "/img_i16.nii", 4, 16, nd, i16.data(), nn * 2, 0.7f, 0.7f, 1.4f, 0.25f, -3.5f);
    write_nifti(out + "/img_f32.nii", 16, 32, nd, f32.data(), nn * 4, -1.0f, 2.0f, 0.0f, 0.0f, 5.0f);
    for (const char *name : {"img_u8", "img_i16", "img_f32"})
        save_raw(load_nifti(out + "/" + name + ".nii"), out + "/" + name + "_expected");
    std::printf("wrote golden io files to %s\n", out.c_str());
    return 0;
}
