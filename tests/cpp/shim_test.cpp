// Compiles the reference-shaped C++ shim (include/convgemm_b200.hpp) the way a
// reference caller would use it, and exercises it. `shim_test` runs the host-only
// checks; `shim_test gpu` also runs conv_gemm / conv_im2col_gemm on the device and
// compares them with a direct seven-loop convolution (conv.hpp:24-55 order).
#include <cmath>
#include <cstdio>
#include <random>

#include "convgemm_b200.hpp"

namespace cg = convgemm_b200;

static int failures = 0;
#define CHECK(c)                                                  \
  do {                                                            \
    if (!(c)) {                                                   \
      std::printf("FAIL %s:%d: %s\n", __FILE__, __LINE__, #c);    \
      ++failures;                                                 \
    }                                                             \
  } while (0)

int main(int argc, char** argv) {
  // geometry (conv_params.hpp:27-43)
  const cg::ConvParams cp{64, 3, 3, 64, 56, 56, 128, 1, 1};
  CHECK(cg::output_dims(cp).h_o == 56 && cg::output_dims(cp).w_o == 56);
  const cg::GemmDims g = cg::gemm_dims(cp);
  CHECK(g.m == 64 && g.n == 401408 && g.k == 576);
  CHECK(cg::im2col_workspace_bytes(cg::ConvParams{192, 5, 5, 64, 55, 55, 1, 1, 0}) == 16646400);
  bool threw = false;
  try {
    cg::output_dims(cg::ConvParams{1, 5, 5, 1, 3, 3, 1, 1, 0});
  } catch (const cg::InvalidGeometry&) {
    threw = true;
  }
  CHECK(threw);
  threw = false;
  try {
    cg::validate(cg::BlockingParams{0, 1, 1, 1, 1});
  } catch (const std::invalid_argument&) {
    threw = true;
  }
  CHECK(threw);
  if (argc > 1 && std::string(argv[1]) == "gpu") {
    const cg::ConvParams c{24, 3, 3, 40, 17, 13, 3, 2, 1};
    std::mt19937_64 rng(101);
    std::uniform_real_distribution<double> u(-1, 1);
    cg::Tensor4<float> F(24, 3, 3, 40), I(17, 13, 40, 3);
    for (cg::index_t i = 0; i < F.size(); ++i) F.data()[i] = (float)u(rng);
    for (cg::index_t i = 0; i < I.size(); ++i) I.data()[i] = (float)u(rng);
    const cg::OutputDims od = cg::output_dims(c);
    // direct conv in double
    std::vector<double> ref((size_t)(24 * od.h_o * od.w_o * 3), 0.0);
    for (cg::index_t b = 0; b < 3; ++b)
      for (cg::index_t ci = 0; ci < 40; ++ci)
        for (cg::index_t iw = 0; iw < od.w_o; ++iw)
          for (cg::index_t ih = 0; ih < od.h_o; ++ih)
            for (cg::index_t kw = 0; kw < 3; ++kw)
              for (cg::index_t kh = 0; kh < 3; ++kh) {
                const cg::index_t h = ih * 2 + kh - 1, w = iw * 2 + kw - 1;
                if (h < 0 || h >= 17 || w < 0 || w >= 13) continue;
                for (cg::index_t k = 0; k < 24; ++k)
                  ref[k + 24 * (ih + od.h_o * (iw + od.w_o * b))] +=
                      (double)F(k, kh, kw, ci) * I(h, w, ci, b);
              }
    for (int algo = 0; algo < 2; ++algo) {
      cg::Tensor4<float> O = algo ? cg::conv_gemm(F, I, c) : cg::conv_im2col_gemm(F, I, c);
      double err = 0, scale = 1;
      for (cg::index_t i = 0; i < O.size(); ++i) {
        err = std::fmax(err, std::fabs(O.data()[i] - ref[i]));
        scale = std::fmax(scale, std::fabs(ref[i]));
      }
      std::printf("%s: normalized max error %.3e\n", algo ? "conv_gemm" : "conv_im2col_gemm", err / scale);
      CHECK(err / scale <= 1e-5);
    }
  }
  std::printf(failures ? "shim_test FAILED\n" : "shim_test OK\n");
  return failures ? 1 : 0;
}
