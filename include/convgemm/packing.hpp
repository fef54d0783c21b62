// convgemm/packing.hpp -- drop-in for proj/include/convgemm/packing.hpp:60-117: the
// right-hand gemm operand abstraction. On the device there are no packed panels; a source
// tells gemm() how the GPU gets the operand (device_operand): a plain matrix is copied as
// is, an Im2colSource becomes the implicit convolution, anything else is read through at().
#pragma once

#include <algorithm>

#include "convgemm/blocking.hpp"
#include "convgemm/scratch.hpp"
#include "convgemm/tensor.hpp"
#include "convgemm/threads.hpp"

namespace convgemm {

struct ConvParams;

namespace detail {
template <typename T>
struct DeviceOperand {
    enum Kind { Elements, Matrix, Conv } kind = Elements;
    MatrixView<const T> matrix{};  // Kind::Matrix
    const T* input = nullptr;      // Kind::Conv: I of the lowered convolution
    const ConvParams* conv = nullptr;
};
}  // namespace detail

template <typename T>
class PackingSource {
public:
    virtual ~PackingSource() = default;
    virtual index_t rows() const = 0;
    virtual index_t cols() const = 0;
    virtual T at(index_t row, index_t col) const = 0;  // pure read
    virtual detail::DeviceOperand<T> device_operand() const { return {}; }
};

// A column-major matrix as the operand (the explicit path's B-hat, fc activations).
template <typename T>
class MatrixSource final : public PackingSource<T> {
public:
    explicit MatrixSource(MatrixView<const T> m) : m_(m) {}
    index_t rows() const override { return m_.rows; }
    index_t cols() const override { return m_.cols; }
    T at(index_t row, index_t col) const override { return m_(row, col); }
    detail::DeviceOperand<T> device_operand() const override {
        detail::DeviceOperand<T> d;
        d.kind = detail::DeviceOperand<T>::Matrix;
        d.matrix = m_;
        return d;
    }

private:
    MatrixView<const T> m_;
};

}  // namespace convgemm
