// blfls_cli.cpp -- command-line front end over the C ABI, mirroring the
// reference CLI's hot-path subcommands (/root/reference/proj/tools/epls_main.cpp):
//
//   blfls smooth [--method blf-ls|nc-ls|ls] [--sigma-s S] [--sigma-r R] [--lambda L]
//                [--pad 16] [--radius r] [--iters k] [--iterations t] [--device d] input output
//   blfls joint  --guide G [same flags] input output
//   blfls convert input output          (raster I/O only, no GPU)
//   blfls texture|clipart [--sigma-s S] [--sigma-r R] [--lambda L] [--n N]
//                [--init-sigma s] [--pad 16] [--device d] input output
//
// texture / clipart are rolling-guidance NC-LS (texture_removal /
// clipart_cleanup, applications.cpp:66-76) with the reference's preparse
// defaults (texture 8 / 0.02, n 3, init 2.5; clipart 6 / 0.02, n 2, init 0.75).
// --method nc-ls filters the gradients with nc_filter, DtParams{sigma_s,
// sigma_r, --iterations (default 3)}.
//
// Defaults follow epls_main.cpp: sigma_s 12, sigma_r 0.04 (joint: 12 / 0.003,
// its preparse defaults), lambda 1024.  Differences: the bilateral stage is
// the brute-force filter (north star) with an explicit --radius (default
// ceil(3 sigma_s) like bilateral.cpp:37); --iters cascades smooth() calls;
// --pad (reflect padding) defaults to 16 as in the reference; --blf grid uses
// the bilateral grid the reference's smooth() runs (default: brute force).
// Image formats: PFM (float, 'Pf' gray / 'PF' RGB, bottom-up, either endian)
// and binary PGM/PPM (P5/P6, 8 or 16 bit), implemented from the Netpbm / PFM
// format definitions with the conventions the reference's CLI tests rely on
// (samples = value / maxval, 8-bit output clamped and rounded).
// PNG / HDR need libpng / the Radiance codec and are not built.
// Exit codes as the reference: 0 ok, 2 usage or invalid argument, 1 other.
#include <algorithm>
#include <cctype>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <iterator>
#include <stdexcept>
#include <string>
#include <vector>

#include "blfls/blfls.hpp"

namespace {

struct UsageError : std::runtime_error {
    using std::runtime_error::runtime_error;
};

// ------------------------------------------------------------ raster I/O --
// Netpbm-family rasters, written from the format definitions:
//   P5 / P6   binary gray / RGB, maxval < 256 one byte per sample, else two
//             bytes big endian; samples map to [0, 1] as value / maxval
//   Pf / PF   float gray / RGB; the third header token is a scale whose sign
//             gives the byte order (negative: little endian); scanlines are
//             stored bottom to top
// Headers are whitespace-separated tokens with '#' comments to end of line,
// followed by exactly one whitespace byte before the sample data.

// The whole file in memory plus a cursor over its header tokens.
class RasterBytes {
public:
    static RasterBytes slurp(const std::string& path)
    {
        std::ifstream in(path, std::ios::binary);
        if (!in) throw std::runtime_error("cannot open '" + path + "'");
        RasterBytes r;
        r.path_ = path;
        r.data_.assign(std::istreambuf_iterator<char>(in), std::istreambuf_iterator<char>());
        return r;
    }
    // next header token (comments skipped); consumes one trailing whitespace byte
    std::string token()
    {
        for (;;) {
            while (pos_ < data_.size() && std::isspace(static_cast<unsigned char>(data_[pos_]))) ++pos_;
            if (pos_ < data_.size() && data_[pos_] == '#') {
                while (pos_ < data_.size() && data_[pos_] != '\n') ++pos_;
                continue;
            }
            break;
        }
        const std::size_t b = pos_;
        while (pos_ < data_.size() && !std::isspace(static_cast<unsigned char>(data_[pos_]))) ++pos_;
        if (b == pos_) throw std::runtime_error("'" + path_ + "': truncated header");
        std::string t = data_.substr(b, pos_ - b);
        if (pos_ < data_.size()) ++pos_;  // the single separator before the payload
        return t;
    }
    long positive(const std::string& what)
    {
        const std::string t = token();
        char* end = nullptr;
        const long v = std::strtol(t.c_str(), &end, 10);
        if (*end != '\0' || v <= 0) throw std::runtime_error("'" + path_ + "': bad " + what + " '" + t + "'");
        return v;
    }
    const unsigned char* payload(std::size_t bytes) const
    {
        if (data_.size() - pos_ < bytes) throw std::runtime_error("'" + path_ + "': truncated sample data");
        return reinterpret_cast<const unsigned char*>(data_.data() + pos_);
    }
    const std::string& path() const { return path_; }

private:
    std::string path_, data_;
    std::size_t pos_ = 0;
};

bool host_is_little_endian()
{
    const uint16_t probe = 1;
    unsigned char b;
    std::memcpy(&b, &probe, 1);
    return b == 1;
}

float float_from_bytes(const unsigned char* p, bool little)
{
    unsigned char b[4];
    if (little == host_is_little_endian())
        std::memcpy(b, p, 4);
    else
        for (int k = 0; k < 4; ++k) b[k] = p[3 - k];
    float v;
    std::memcpy(&v, b, 4);
    return v;
}

blfls::Image decode_raster(RasterBytes& r)
{
    const std::string magic = r.token();
    const bool is_float = magic == "Pf" || magic == "PF";
    const bool is_int = magic == "P5" || magic == "P6";
    if (!is_float && !is_int)
        throw std::runtime_error("'" + r.path() + "': not a PFM / binary PGM / binary PPM file");
    const int ch = (magic == "PF" || magic == "P6") ? 3 : 1;
    const int w = static_cast<int>(r.positive("width"));
    const int h = static_cast<int>(r.positive("height"));
    blfls::Image img(w, h, ch);
    const std::size_t samples = static_cast<std::size_t>(w) * h * ch;
    if (is_float) {
        const std::string st = r.token();
        char* end = nullptr;
        const double scale = std::strtod(st.c_str(), &end);
        if (*end != '\0' || scale == 0.0 || !std::isfinite(scale))
            throw std::runtime_error("'" + r.path() + "': bad PFM scale '" + st + "'");
        const unsigned char* p = r.payload(samples * 4);
        const bool little = scale < 0.0;
        for (int row = 0; row < h; ++row) {          // file row 0 is the bottom scanline
            const int y = h - 1 - row;
            for (int x = 0; x < w; ++x)
                for (int c = 0; c < ch; ++c, p += 4) img.at(c, y, x) = float_from_bytes(p, little);
        }
    } else {
        const long maxval = r.positive("maxval");
        if (maxval > 65535) throw std::runtime_error("'" + r.path() + "': maxval above 65535");
        const int width_bytes = maxval > 255 ? 2 : 1;
        const unsigned char* p = r.payload(samples * width_bytes);
        const double inv = 1.0 / static_cast<double>(maxval);
        for (int y = 0; y < h; ++y)
            for (int x = 0; x < w; ++x)
                for (int c = 0; c < ch; ++c) {
                    const unsigned v = width_bytes == 2 ? (unsigned(p[0]) << 8) | p[1] : p[0];
                    p += width_bytes;
                    img.at(c, y, x) = v * inv;
                }
    }
    return img;
}

void write_bytes(const std::string& path, const std::string& header, const std::vector<unsigned char>& body)
{
    std::ofstream out(path, std::ios::binary | std::ios::trunc);
    if (!out) throw std::runtime_error("cannot open '" + path + "' for writing");
    out.write(header.data(), static_cast<std::streamsize>(header.size()));
    out.write(reinterpret_cast<const char*>(body.data()), static_cast<std::streamsize>(body.size()));
    if (!out) throw std::runtime_error("'" + path + "': write failed");
}

// PFM out: host byte order, declared by the sign of the scale
void encode_float_raster(const std::string& path, const blfls::Image& img)
{
    const int w = img.width(), h = img.height(), ch = img.channels();
    const bool little = host_is_little_endian();
    const std::string header = std::string(ch == 3 ? "PF" : "Pf") + "\n" + std::to_string(w) + " " +
                               std::to_string(h) + "\n" + (little ? "-1.0" : "1.0") + "\n";
    std::vector<unsigned char> body(static_cast<std::size_t>(w) * h * ch * 4);
    unsigned char* p = body.data();
    for (int y = h - 1; y >= 0; --y)
        for (int x = 0; x < w; ++x)
            for (int c = 0; c < ch; ++c, p += 4) {
                const float v = static_cast<float>(img.at(c, y, x));
                std::memcpy(p, &v, 4);
            }
    write_bytes(path, header, body);
}

// PGM / PPM out: 8-bit, samples clamped to [0, 1] and rounded to nearest
void encode_byte_raster(const std::string& path, const blfls::Image& img)
{
    const int w = img.width(), h = img.height(), ch = img.channels();
    const std::string header = std::string(ch == 3 ? "P6" : "P5") + "\n" + std::to_string(w) + " " +
                               std::to_string(h) + "\n255\n";
    std::vector<unsigned char> body;
    body.reserve(static_cast<std::size_t>(w) * h * ch);
    for (int y = 0; y < h; ++y)
        for (int x = 0; x < w; ++x)
            for (int c = 0; c < ch; ++c) {
                const double v = img.at(c, y, x);
                const double q = std::floor((v < 0.0 ? 0.0 : (v > 1.0 ? 1.0 : v)) * 255.0 + 0.5);
                body.push_back(static_cast<unsigned char>(q));
            }
    write_bytes(path, header, body);
}

std::string lower_extension(const std::string& path)
{
    const auto dot = path.find_last_of('.');
    std::string e = dot == std::string::npos ? std::string() : path.substr(dot + 1);
    std::transform(e.begin(), e.end(), e.begin(), [](unsigned char c) { return static_cast<char>(std::tolower(c)); });
    return e;
}

blfls::Image load_image(const std::string& path)
{
    const std::string e = lower_extension(path);
    if (e != "pfm" && e != "pgm" && e != "ppm")
        throw std::runtime_error("'" + path + "': unsupported image extension ." + e +
                                 " (this build reads .pfm/.pgm/.ppm)");
    RasterBytes r = RasterBytes::slurp(path);
    return decode_raster(r);
}

void save_image(const std::string& path, const blfls::Image& img)
{
    const std::string e = lower_extension(path);
    if (e == "pfm") return encode_float_raster(path, img);
    if (e == "pgm" || e == "ppm") return encode_byte_raster(path, img);
    throw std::runtime_error("'" + path + "': unsupported image extension ." + e +
                             " (this build writes .pfm/.pgm/.ppm)");
}

struct Options {
    std::string cmd, input, output, guide, method = "blf-ls";
    double sigma_s = 12.0, sigma_r = 0.04, lambda = -1.0, init_sigma = 2.5;
    int pad = 16, radius = -1, iters = 1, device = 0, backend = BLFLS_BACKEND_BRUTE;
    int iterations = 3, n = 3;
};

double parse_double(const std::string& flag, const char* v)
{
    char* end = nullptr;
    const double d = std::strtod(v, &end);
    if (!end || *end || !std::isfinite(d)) throw UsageError(flag + ": not a number: " + v);
    return d;
}

int parse_int(const std::string& flag, const char* v)
{
    char* end = nullptr;
    const long d = std::strtol(v, &end, 10);
    if (!end || *end) throw UsageError(flag + ": not an integer: " + v);
    return static_cast<int>(d);
}

Options parse(int argc, char** argv)
{
    if (argc < 2) throw UsageError("a subcommand is required: smooth | joint | texture | clipart | convert");
    Options o;
    o.cmd = argv[1];
    if (o.cmd != "smooth" && o.cmd != "joint" && o.cmd != "texture" && o.cmd != "clipart" && o.cmd != "convert")
        throw UsageError("unknown subcommand '" + o.cmd + "'");
    const bool rolling = o.cmd == "texture" || o.cmd == "clipart";
    if (o.cmd == "joint") {  // epls_main.cpp preparse defaults of `joint`
        o.sigma_s = 12.0;
        o.sigma_r = 0.003;
    } else if (o.cmd == "texture") {  // ... of `texture`
        o.sigma_s = 8.0;
        o.sigma_r = 0.02;
        o.n = 3;
        o.init_sigma = 2.5;
    } else if (o.cmd == "clipart") {  // ... of `clipart`
        o.sigma_s = 6.0;
        o.sigma_r = 0.02;
        o.n = 2;
        o.init_sigma = 0.75;
    }
    std::vector<std::string> pos;
    for (int i = 2; i < argc; ++i) {
        const std::string a = argv[i];
        auto next = [&]() -> const char* {
            if (i + 1 >= argc) throw UsageError(a + " needs a value");
            return argv[++i];
        };
        if (a == "--method" && !rolling) {
            o.method = next();
            if (o.method != "blf-ls" && o.method != "nc-ls" && o.method != "ls")
                throw UsageError("--method: GPU build supports blf-ls, nc-ls and ls, got '" + o.method + "'");
        } else if (a == "--sigma-s") {
            o.sigma_s = parse_double(a, next());
            if (!(o.sigma_s > 0)) throw UsageError("--sigma-s must be positive");
        } else if (a == "--sigma-r") {
            o.sigma_r = parse_double(a, next());
            if (!(o.sigma_r > 0)) throw UsageError("--sigma-r must be positive");
        } else if (a == "--lambda") {
            o.lambda = parse_double(a, next());
        } else if (a == "--pad") {
            o.pad = parse_int(a, next());
            if (o.pad < 0) throw UsageError("--pad must be non-negative");
        } else if (a == "--radius") {
            o.radius = parse_int(a, next());
        } else if (a == "--iters") {
            o.iters = parse_int(a, next());
            if (o.iters < 1) throw UsageError("--iters must be >= 1");
        } else if (a == "--iterations" && !rolling) {
            o.iterations = parse_int(a, next());  // DtParams::iterations (nc-ls)
            if (o.iterations < 1) throw UsageError("--iterations must be positive");
        } else if (a == "--n" && rolling) {
            o.n = parse_int(a, next());
            if (o.n < 1) throw UsageError("--n must be positive");
        } else if (a == "--init-sigma" && rolling) {
            o.init_sigma = parse_double(a, next());
            if (!(o.init_sigma > 0)) throw UsageError("--init-sigma must be positive");
        } else if (a == "--blf") {
            const std::string b = next();
            if (b == "grid") o.backend = BLFLS_BACKEND_GRID;
            else if (b == "brute") o.backend = BLFLS_BACKEND_BRUTE;
            else throw UsageError("--blf: brute or grid, got '" + b + "'");
        } else if (a == "--device") {
            o.device = parse_int(a, next());
        } else if (a == "--guide" && o.cmd == "joint") {
            o.guide = next();
        } else if (a == "--threads") {
            next();  // host thread count of the reference; the GPU path ignores it
        } else if (!a.empty() && a[0] == '-' && a.size() > 1) {
            throw UsageError("unknown option " + a);
        } else {
            pos.push_back(a);
        }
    }
    if (pos.size() != 2) throw UsageError("expected: input output");
    if (o.cmd == "joint" && o.guide.empty()) throw UsageError("joint: --guide is required");
    o.input = pos[0];
    o.output = pos[1];
    return o;
}

int run(const Options& o)
{
    const blfls::Image in = load_image(o.input);
    if (o.cmd == "convert") {  // raster I/O only (no device): format conversion
        save_image(o.output, in);
        return 0;
    }
    const double lam = o.lambda >= 0.0 ? o.lambda : 1024.0;
    const blfls::DtParams dt{o.sigma_s, o.sigma_r, o.iterations};
    blfls::Image out;
    if (o.cmd == "texture" || o.cmd == "clipart") {
        out = blfls::rolling_nc_ls(in, dt, blfls::SolveParams{lam, o.pad},
                                   blfls::RollingParams{o.n, o.init_sigma}, o.device);
    } else if (o.method == "nc-ls") {
        blfls::Image guide;
        if (o.cmd == "joint") {
            guide = load_image(o.guide);
            if (!guide.same_shape(in)) throw std::invalid_argument("flash_no_flash: image shapes differ");
        }
        out = blfls::nc_ls(in, o.cmd == "joint" ? &guide : nullptr, lam, dt, o.iters, o.device, o.pad);
    } else if (o.method == "ls") {
        blfls::Image zero(in.width(), in.height(), in.channels(), 0.0);
        // plain LS == lsgrad with a zero target (test_solver.cpp:129-134); the
        // reference normalises first (pipelines.cpp:64-68), a no-op for this
        // affine-equivariant solve
        out = blfls::lsgrad_solve_fft(in, zero, zero, lam, o.device, o.pad);
    } else if (o.cmd == "joint") {
        const blfls::Image guide = load_image(o.guide);
        if (guide.width() != in.width() || guide.height() != in.height())
            throw std::invalid_argument("flash_no_flash: image shapes differ");
        out = blfls::blf_ls(in, &guide, lam, o.sigma_s, o.sigma_r, o.iters, o.radius, o.device, o.pad,
                            o.backend);
    } else {
        out = blfls::blf_ls(in, nullptr, lam, o.sigma_s, o.sigma_r, o.iters, o.radius, o.device, o.pad,
                            o.backend);
    }
    save_image(o.output, out);
    return 0;
}

}  // namespace

int main(int argc, char** argv)
{
    Options o;
    try {
        o = parse(argc, argv);
    } catch (const UsageError& e) {
        std::fprintf(stderr, "usage error: %s\n", e.what());
        return 2;
    }
    try {
        return run(o);
    } catch (const std::invalid_argument& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    } catch (const std::domain_error& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 2;
    } catch (const std::exception& e) {
        std::fprintf(stderr, "error: %s\n", e.what());
        return 1;
    }
}
