// _swarmsim_b200 — the codec / cost-model half of the reference's Python
// module (P/bindings/module.cpp:17-23, 35-53, 143-163) with identical names,
// argument names, defaults and exception mapping (ConfigError -> ValueError
// subclass), backed by the B200 implementation in libswarm_b200.so.
#include <pybind11/pybind11.h>
#include <pybind11/stl.h>

#include "swarm_b200.h"
#include "swarmsim/compression.hpp"
#include "swarmsim/cost_model.hpp"
#include "swarmsim/errors.hpp"

namespace py = pybind11;
using namespace swarmsim;

PYBIND11_MODULE(_swarmsim_b200, m) {
    m.doc() = "SWARM per-stage hot path on B200: int8 boundary codec, maxout, LayerNorm";

    py::register_exception<ConfigError>(m, "ConfigError", PyExc_ValueError);
    py::register_exception<ParseError>(m, "ParseError", PyExc_ValueError);
    py::register_exception<NoPeerAvailable>(m, "NoPeerAvailable", PyExc_RuntimeError);

    py::class_<cost_model::LayerShape>(m, "LayerShape")
        .def(py::init<>())
        .def_readwrite("d_model", &cost_model::LayerShape::d_model)
        .def_readwrite("d_ffn", &cost_model::LayerShape::d_ffn)
        .def_readwrite("n_heads", &cost_model::LayerShape::n_heads)
        .def_readwrite("seq_len", &cost_model::LayerShape::seq_len)
        .def_readwrite("batch", &cost_model::LayerShape::batch)
        .def_readwrite("layers_per_stage", &cost_model::LayerShape::layers_per_stage)
        .def_readwrite("activation_bytes_per_element", &cost_model::LayerShape::activation_bytes_per_element);

    m.def("params_per_layer", &cost_model::params_per_layer, py::arg("shape"));
    m.def("flops_per_stage", &cost_model::flops_per_stage, py::arg("shape"), py::arg("include_backward"));
    m.def("activation_payload_bits", &cost_model::activation_payload_bits, py::arg("shape"));
    py::class_<cost_model::DeviceProfile>(m, "DeviceProfile")
        .def(py::init<>())
        .def_readwrite("effective_flops", &cost_model::DeviceProfile::effective_flops)
        .def_readwrite("upload_bps", &cost_model::DeviceProfile::upload_bps)
        .def_readwrite("download_bps", &cost_model::DeviceProfile::download_bps)
        .def_readwrite("rtt_seconds", &cost_model::DeviceProfile::rtt_seconds);
    py::class_<cost_model::CostBreakdown>(m, "CostBreakdown")
        .def(py::init<>())
        .def_readonly("compute_seconds", &cost_model::CostBreakdown::compute_seconds)
        .def_readonly("comm_seconds", &cost_model::CostBreakdown::comm_seconds)
        .def_readonly("total_seconds", &cost_model::CostBreakdown::total_seconds)
        .def_readonly("idle_fraction", &cost_model::CostBreakdown::idle_fraction)
        .def_readonly("utilization", &cost_model::CostBreakdown::utilization);
    m.def("stage_cost", &cost_model::stage_cost, py::arg("shape"), py::arg("device"), py::arg("overlap") = true);
    m.def("square_cube_ratio", &cost_model::square_cube_ratio, py::arg("shape"));
    m.def("calibrated_profile", &cost_model::calibrated_profile, py::arg("shape"), py::arg("measured_visit_seconds"),
          py::arg("link_bps"), py::arg("link_rtt_seconds") = 0.0);
    m.def("preset", &cost_model::preset, py::arg("name"));
    m.def("preset_names", &cost_model::preset_names);

    py::class_<compress::QuantizedTensor>(m, "QuantizedTensor")
        .def(py::init<>())
        .def_readonly("codes", &compress::QuantizedTensor::codes)
        .def_readonly("absmax", &compress::QuantizedTensor::absmax)
        .def_readonly("block_size", &compress::QuantizedTensor::block_size)
        .def("payload_bits", &compress::QuantizedTensor::payload_bits);

    m.def("quantize_blockwise", &compress::quantize_blockwise, py::arg("x"), py::arg("block_size") = 2048);
    m.def("dequantize_blockwise", &compress::dequantize_blockwise, py::arg("q"));
    m.def("maxout_k", &compress::maxout_k, py::arg("x"), py::arg("k"));
    m.def(
        "layer_norm", [](const std::vector<double>& x) { return compress::layer_norm(x); }, py::arg("x"));
    m.def(
        "compressed_payload_bits",
        [](const cost_model::LayerShape& shape, const std::string& kind, double factor) {
            return compress::payload_bits(shape, {compress::kind_from_name(kind), factor});
        },
        py::arg("shape"), py::arg("kind"), py::arg("factor") = 1.0);

    // additive: the bottleneck pair, which the reference binds only in C++
    m.def("bottleneck_forward",
          [](const std::vector<double>& x, const std::vector<std::vector<double>>& w_c, double epsilon) {
              compress::LayerNormParams p;
              p.epsilon = epsilon;
              return compress::bottleneck_forward(x, w_c, p);
          },
          py::arg("x"), py::arg("w_c"), py::arg("epsilon") = 1e-5);
    m.def("bottleneck_decompress", &compress::bottleneck_decompress, py::arg("y"), py::arg("w_d"));
    m.def("launch_count", &swarm_launch_count);
}
