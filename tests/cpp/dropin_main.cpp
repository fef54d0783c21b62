// Drives the REFERENCE's own simulator sources (proj/src/bench.cpp and model.cpp,
// compiled unchanged against include/convgemm/ by tests/test_cpp_dropin.py) on the B200
// operator: every algorithm over a small model, with the reference's per-layer check
// against conv_direct switched on (bench.cpp:227-233: normalised max error <= 1e-5,
// throws on failure), then its CSV writer.
#include <cstdio>
#include <iostream>
#include <sstream>

#include "convgemm/bench.hpp"
#include "convgemm/conv.hpp"

int main() {
    using namespace convgemm;
    std::istringstream text(
        "# tiny test model\n"
        "conv 16 3 3 3 20 20 1 1\n"
        "pool 10 10 16\n"
        "conv 32 3 3 16 10 10 2 1\n"
        "conv 24 1 1 32 5 5 1 0\n"
        "fc 10 600\n");
    const ModelSpec model = parse_model(text, "tiny");
    std::printf("model %s: %lld layers, %lld conv, workspace(b=2) %lld bytes\n", model.name.c_str(),
                (long long)model.layers.size(), (long long)model.count(LayerSpec::Kind::Conv),
                (long long)model_workspace_bytes(model, 2));
    write_csv_header(std::cout);
    for (Algo algo : {Algo::Direct, Algo::Im2col, Algo::ConvGemm, Algo::GemmOnly, Algo::Im2colOnly}) {
        RunOptions opt;
        opt.min_time = 0.0;
        opt.check = true;  // every conv output checked against conv_direct<float>
        const std::vector<LayerResult> rows = run_inference(model, 2, algo, opt);
        write_csv_rows(std::cout, model, 2, algo, opt.threads, rows);
    }
    std::printf("dropin OK\n");
    return 0;
}
