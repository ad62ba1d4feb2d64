// File formats of the online phase's inputs (SURVEY §8b loaders, §8f-2):
//   * matrix CSV  <- read_matrix_csv / write_matrix_csv (core.cpp:191-254):
//     header "app,c<CPU>_g<GPU>,...", one row per app, empty cell = unobserved,
//     values in shortest round-trip decimal (format_double, core.cpp:171-175);
//   * binary CSR  (no reference counterpart: CSV at C2 is tens of GB of text) —
//     the same matrix as a little-endian header + CSR arrays + app ids;
//   * predictor model file <- pred::load_predictor / predictor_from_json
//     (predictor.cpp:301-331) over nn::model_from_json (nnkit.cpp:332-365).
// Host-only code; validation and error kinds follow the reference:
// missing_artifact_error -> OCG_E_MISSING, config_error / invalid_argument ->
// OCG_E_INVALID, runtime_error ("model file: ...") -> OCG_E_LOGIC.
#include <algorithm>
#include <charconv>
#include <cmath>
#include <cstdint>
#include <cstring>
#include <fstream>
#include <memory>
#include <set>
#include <sstream>
#include <string>
#include <vector>

#include "../../include/ocg.h"
#include <nlohmann/json.hpp>

int ocg_internal_fail(int code, const std::string& msg);

struct ocg_matrix {
    std::vector<std::string> apps;
    std::vector<int32_t> cpu, gpu;  // per column
    std::vector<int64_t> rp;
    std::vector<int32_t> col;
    std::vector<double> val;
};

namespace {

int fail(int code, const std::string& msg) { return ocg_internal_fail(code, msg); }

std::string format_double(double v) {  // core.cpp:171-175
    char buf[32];
    const auto res = std::to_chars(buf, buf + sizeof(buf), v);
    return std::string(buf, res.ptr);
}

std::vector<std::string> split_csv_line(const std::string& line) {  // core.cpp:177-189
    std::vector<std::string> cells;
    std::string cur;
    for (const char ch : line) {
        if (ch == ',') {
            cells.push_back(std::move(cur));
            cur.clear();
        } else if (ch != '\r') {
            cur.push_back(ch);
        }
    }
    cells.push_back(std::move(cur));
    return cells;
}

bool parse_setting_label(const std::string& label, int32_t& cpu, int32_t& gpu) {  // core.cpp:20-34
    if (label.size() < 4 || label[0] != 'c') return false;
    const auto sep = label.find("_g");
    if (sep == std::string::npos || sep == 1 || sep + 2 >= label.size()) return false;
    const char* cb = label.data() + 1;
    const char* ce = label.data() + sep;
    const char* gb = label.data() + sep + 2;
    const char* ge = label.data() + label.size();
    int c = 0, g = 0;
    auto rc = std::from_chars(cb, ce, c);
    auto rg = std::from_chars(gb, ge, g);
    if (rc.ec != std::errc{} || rc.ptr != ce || rg.ec != std::errc{} || rg.ptr != ge) return false;
    if (c <= 0 || g <= 0) return false;
    cpu = c;
    gpu = g;
    return true;
}

// PerformanceMatrix ctor checks (core.cpp:84-111)
int check_matrix_ids(const std::vector<std::string>& ids, const std::vector<int32_t>& cpu,
                     const std::vector<int32_t>& gpu) {
    if (ids.empty()) return fail(OCG_E_INVALID, "app id list is empty");
    std::set<std::string> seen;
    for (const auto& id : ids) {
        if (id.empty()) return fail(OCG_E_INVALID, "empty app id");
        if (id.find_first_of(",\n\r") != std::string::npos)
            return fail(OCG_E_INVALID, "app id contains csv delimiter: " + id);
        if (!seen.insert(id).second) return fail(OCG_E_INVALID, "duplicate app id: " + id);
    }
    if (cpu.empty()) return fail(OCG_E_INVALID, "empty setting list");
    std::set<std::pair<int32_t, int32_t>> ss;
    for (size_t j = 0; j < cpu.size(); ++j)
        if (!ss.insert({cpu[j], gpu[j]}).second) return fail(OCG_E_INVALID, "duplicate setting");
    return OCG_OK;
}

bool valid_value(double v) { return std::isfinite(v) && v > 0.0 && v <= 1.25; }  // core.cpp:144-146

// ------------------------------------------------------------ predictor
struct PredModel {
    std::vector<int64_t> dims;
    std::vector<int32_t> acts;
    std::vector<double> params;
    double mean[7] = {}, sd[7] = {};
    bool has_stats = false;
};

int parse_predictor(const char* text, PredModel& pm) {
    nlohmann::json doc;
    try {
        doc = nlohmann::json::parse(text);
    } catch (const nlohmann::json::exception& e) {
        return fail(OCG_E_LOGIC, std::string("model file: bad json: ") + e.what());
    }
    try {
        if (!doc.contains("format_version") || doc["format_version"].get<int>() != 1)
            return fail(OCG_E_LOGIC, "model file: unsupported format_version");
        const auto dims = doc.at("architecture").at("dims").get<std::vector<std::size_t>>();
        const auto acts = doc.at("architecture").at("activations").get<std::vector<std::string>>();
        if (dims.size() < 2 || acts.size() != dims.size() - 1)
            return fail(OCG_E_LOGIC, "model file: inconsistent architecture");
        const auto& jl = doc.at("layers");
        if (jl.size() != acts.size()) return fail(OCG_E_LOGIC, "model file: layer count mismatch");
        pm.dims.assign(dims.begin(), dims.end());
        for (size_t l = 0; l < jl.size(); ++l) {
            const std::string& a = acts[l];  // nn::parse_activation (nnkit.cpp:20-25)
            if (a == "selu") pm.acts.push_back(0);
            else if (a == "relu") pm.acts.push_back(1);
            else if (a == "identity") pm.acts.push_back(2);
            else return fail(OCG_E_INVALID, "unknown activation: " + a);
            const auto& weights = jl[l].at("weights");
            if (weights.size() != dims[l + 1]) return fail(OCG_E_LOGIC, "model file: weight shape");
            for (const auto& row : weights) {
                if (row.size() != dims[l]) return fail(OCG_E_LOGIC, "model file: weight shape");
                for (const auto& v : row) pm.params.push_back(v.get<double>());
            }
            const auto b = jl[l].at("biases").get<std::vector<double>>();
            if (b.size() != dims[l + 1]) return fail(OCG_E_LOGIC, "model file: bias shape");
            pm.params.insert(pm.params.end(), b.begin(), b.end());
        }
        for (const double p : pm.params)  // MlpModel::check_finite (nnkit.cpp:106-113)
            if (!std::isfinite(p)) return fail(OCG_E_LOGIC, "non-finite weight");
        if (doc.contains("feature_stats")) {  // predictor.cpp:305-314
            const auto mean = doc["feature_stats"].at("mean").get<std::vector<double>>();
            const auto sd = doc["feature_stats"].at("std").get<std::vector<double>>();
            if (mean.size() != 7 || sd.size() != 7)
                return fail(OCG_E_LOGIC, "predictor model: feature_stats shape mismatch");
            std::copy(mean.begin(), mean.end(), pm.mean);
            std::copy(sd.begin(), sd.end(), pm.sd);
            pm.has_stats = true;
        }
    } catch (const nlohmann::json::exception& e) {
        return fail(OCG_E_LOGIC, std::string("model file: ") + e.what());
    }
    return OCG_OK;
}

int read_file(const char* path, std::string& out, const char* what) {
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(OCG_E_MISSING, std::string("missing ") + what + ": " + path);
    std::ostringstream buf;
    buf << f.rdbuf();
    out = buf.str();
    return OCG_OK;
}

constexpr char kBinMagic[8] = {'O', 'C', 'G', 'C', 'S', 'R', '1', '\0'};

}  // namespace

extern "C" {

// ------------------------------------------------------------ matrices
int ocg_matrix_read_csv(const char* path, ocg_matrix** out) {
    if (!path || !out) return fail(OCG_E_INVALID, "null argument");
    *out = nullptr;
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(OCG_E_MISSING, std::string("missing matrix csv: ") + path);  // core.cpp:252
    std::string line;
    if (!std::getline(f, line)) return fail(OCG_E_INVALID, "matrix csv: empty file");
    const auto header = split_csv_line(line);
    if (header.empty() || header[0] != "app") return fail(OCG_E_INVALID, "matrix csv: header must start with 'app'");
    if (header.size() < 2) return fail(OCG_E_INVALID, "matrix csv: no setting columns");
    auto M = std::make_unique<ocg_matrix>();
    for (size_t j = 1; j < header.size(); ++j) {
        int32_t c = 0, g = 0;
        if (!parse_setting_label(header[j], c, g))
            return fail(OCG_E_INVALID, "matrix csv: bad setting label '" + header[j] + "'");
        M->cpu.push_back(c);
        M->gpu.push_back(g);
    }
    std::vector<std::vector<std::string>> rows;
    while (std::getline(f, line)) {
        if (line.empty()) continue;
        auto cells = split_csv_line(line);
        if (cells.size() != header.size())
            return fail(OCG_E_INVALID, "matrix csv: ragged row for '" + (cells.empty() ? "" : cells[0]) + "'");
        M->apps.push_back(cells[0]);
        rows.push_back(std::move(cells));
    }
    int rc = check_matrix_ids(M->apps, M->cpu, M->gpu);
    if (rc) return rc;
    const size_t n = M->cpu.size();
    M->rp.assign(rows.size() + 1, 0);
    for (size_t i = 0; i < rows.size(); ++i) {
        for (size_t j = 0; j < n; ++j) {
            const std::string& cell = rows[i][j + 1];
            if (cell.empty()) continue;
            double v = 0.0;
            const auto res = std::from_chars(cell.data(), cell.data() + cell.size(), v);
            if (res.ec != std::errc{} || res.ptr != cell.data() + cell.size())
                return fail(OCG_E_INVALID, "matrix csv: non-numeric cell '" + cell + "'");
            if (!valid_value(v)) return fail(OCG_E_INVALID, "normalized performance outside (0, 1.25]: " + format_double(v));
            M->col.push_back(static_cast<int32_t>(j));
            M->val.push_back(v);
        }
        M->rp[i + 1] = static_cast<int64_t>(M->col.size());
    }
    *out = M.release();
    return OCG_OK;
}

int ocg_matrix_create(int64_t m, int64_t n, const char* const* app_ids, const int32_t* cpu, const int32_t* gpu,
                      const int64_t* row_ptr, const int32_t* col, const double* val, ocg_matrix** out) {
    if (!out || !app_ids || !cpu || !gpu || !row_ptr || (row_ptr[m] > 0 && (!col || !val)))
        return fail(OCG_E_INVALID, "null argument");
    *out = nullptr;
    if (m < 0 || n <= 0) return fail(OCG_E_INVALID, "bad matrix shape");
    auto M = std::make_unique<ocg_matrix>();
    for (int64_t i = 0; i < m; ++i) M->apps.emplace_back(app_ids[i] ? app_ids[i] : "");
    M->cpu.assign(cpu, cpu + n);
    M->gpu.assign(gpu, gpu + n);
    for (int64_t j = 0; j < n; ++j)
        if (cpu[j] <= 0 || gpu[j] <= 0) return fail(OCG_E_INVALID, "caps must be positive watts");
    int rc = check_matrix_ids(M->apps, M->cpu, M->gpu);
    if (rc) return rc;
    if (row_ptr[0] != 0) return fail(OCG_E_INVALID, "csr: row_ptr[0] must be 0");
    for (int64_t i = 0; i < m; ++i) {
        if (row_ptr[i + 1] < row_ptr[i]) return fail(OCG_E_INVALID, "csr: row_ptr must be non-decreasing");
        for (int64_t q = row_ptr[i]; q < row_ptr[i + 1]; ++q) {
            if (col[q] < 0 || col[q] >= n) return fail(OCG_E_RANGE, "matrix index out of range");
            if (q > row_ptr[i] && col[q - 1] >= col[q])
                return fail(OCG_E_INVALID, "csr: columns must be strictly ascending within a row");
            if (!valid_value(val[q]))
                return fail(OCG_E_INVALID, "normalized performance outside (0, 1.25]: " + format_double(val[q]));
        }
    }
    M->rp.assign(row_ptr, row_ptr + m + 1);
    M->col.assign(col, col + row_ptr[m]);
    M->val.assign(val, val + row_ptr[m]);
    *out = M.release();
    return OCG_OK;
}

int ocg_matrix_write_csv(const ocg_matrix* M, const char* path) {
    if (!M || !path) return fail(OCG_E_INVALID, "null argument");
    std::ofstream f(path, std::ios::binary);
    if (!f) return fail(OCG_E_LOGIC, std::string("cannot open for writing: ") + path);
    std::string buf = "app";
    for (size_t j = 0; j < M->cpu.size(); ++j)
        buf += ",c" + std::to_string(M->cpu[j]) + "_g" + std::to_string(M->gpu[j]);
    buf += '\n';
    const size_t n = M->cpu.size();
    for (size_t i = 0; i < M->apps.size(); ++i) {
        buf += M->apps[i];
        int64_t q = M->rp[i];
        for (size_t j = 0; j < n; ++j) {
            buf += ',';
            if (q < M->rp[i + 1] && static_cast<size_t>(M->col[static_cast<size_t>(q)]) == j)
                buf += format_double(M->val[static_cast<size_t>(q++)]);
        }
        buf += '\n';
        if (buf.size() > (size_t(1) << 24)) {
            f << buf;
            buf.clear();
        }
    }
    f << buf;
    return f ? OCG_OK : fail(OCG_E_LOGIC, std::string("write failed: ") + path);
}

int ocg_matrix_shape(const ocg_matrix* M, int64_t* m, int64_t* n, int64_t* nnz) {
    if (!M) return fail(OCG_E_INVALID, "null matrix");
    if (m) *m = static_cast<int64_t>(M->apps.size());
    if (n) *n = static_cast<int64_t>(M->cpu.size());
    if (nnz) *nnz = static_cast<int64_t>(M->col.size());
    return OCG_OK;
}

int ocg_matrix_get(const ocg_matrix* M, int32_t* cpu, int32_t* gpu, int64_t* row_ptr, int32_t* col, double* val) {
    if (!M) return fail(OCG_E_INVALID, "null matrix");
    if (cpu) std::copy(M->cpu.begin(), M->cpu.end(), cpu);
    if (gpu) std::copy(M->gpu.begin(), M->gpu.end(), gpu);
    if (row_ptr) std::copy(M->rp.begin(), M->rp.end(), row_ptr);
    if (col) std::copy(M->col.begin(), M->col.end(), col);
    if (val) std::copy(M->val.begin(), M->val.end(), val);
    return OCG_OK;
}

const char* ocg_matrix_app_id(const ocg_matrix* M, int64_t i) {
    if (!M || i < 0 || i >= static_cast<int64_t>(M->apps.size())) return nullptr;
    return M->apps[static_cast<size_t>(i)].c_str();
}

int ocg_matrix_save_bin(const ocg_matrix* M, const char* path) {
    if (!M || !path) return fail(OCG_E_INVALID, "null argument");
    std::ofstream f(path, std::ios::binary);
    if (!f) return fail(OCG_E_LOGIC, std::string("cannot open for writing: ") + path);
    const int64_t hdr[3] = {static_cast<int64_t>(M->apps.size()), static_cast<int64_t>(M->cpu.size()),
                            static_cast<int64_t>(M->col.size())};
    f.write(kBinMagic, 8);
    f.write(reinterpret_cast<const char*>(hdr), sizeof hdr);
    f.write(reinterpret_cast<const char*>(M->cpu.data()), sizeof(int32_t) * M->cpu.size());
    f.write(reinterpret_cast<const char*>(M->gpu.data()), sizeof(int32_t) * M->gpu.size());
    f.write(reinterpret_cast<const char*>(M->rp.data()), sizeof(int64_t) * M->rp.size());
    f.write(reinterpret_cast<const char*>(M->col.data()), sizeof(int32_t) * M->col.size());
    f.write(reinterpret_cast<const char*>(M->val.data()), sizeof(double) * M->val.size());
    for (const auto& a : M->apps) {
        const uint32_t len = static_cast<uint32_t>(a.size());
        f.write(reinterpret_cast<const char*>(&len), 4);
        f.write(a.data(), len);
    }
    return f ? OCG_OK : fail(OCG_E_LOGIC, std::string("write failed: ") + path);
}

int ocg_matrix_load_bin(const char* path, ocg_matrix** out) {
    if (!path || !out) return fail(OCG_E_INVALID, "null argument");
    *out = nullptr;
    std::ifstream f(path, std::ios::binary);
    if (!f) return fail(OCG_E_MISSING, std::string("missing matrix file: ") + path);
    char magic[8];
    int64_t hdr[3];
    if (!f.read(magic, 8) || std::memcmp(magic, kBinMagic, 8) != 0)
        return fail(OCG_E_INVALID, "matrix file: bad magic (not an OCGCSR1 file)");
    if (!f.read(reinterpret_cast<char*>(hdr), sizeof hdr) || hdr[0] < 0 || hdr[1] <= 0 || hdr[2] < 0)
        return fail(OCG_E_INVALID, "matrix file: bad header");
    const int64_t m = hdr[0], n = hdr[1], nnz = hdr[2];
    auto M = std::make_unique<ocg_matrix>();
    M->cpu.resize(static_cast<size_t>(n));
    M->gpu.resize(static_cast<size_t>(n));
    M->rp.resize(static_cast<size_t>(m + 1));
    M->col.resize(static_cast<size_t>(nnz));
    M->val.resize(static_cast<size_t>(nnz));
    f.read(reinterpret_cast<char*>(M->cpu.data()), sizeof(int32_t) * n);
    f.read(reinterpret_cast<char*>(M->gpu.data()), sizeof(int32_t) * n);
    f.read(reinterpret_cast<char*>(M->rp.data()), sizeof(int64_t) * (m + 1));
    f.read(reinterpret_cast<char*>(M->col.data()), sizeof(int32_t) * nnz);
    f.read(reinterpret_cast<char*>(M->val.data()), sizeof(double) * nnz);
    for (int64_t i = 0; i < m && f; ++i) {
        uint32_t len = 0;
        f.read(reinterpret_cast<char*>(&len), 4);
        std::string a(len, '\0');
        f.read(a.data(), len);
        M->apps.push_back(std::move(a));
    }
    if (!f) return fail(OCG_E_INVALID, "matrix file: truncated");
    std::vector<const char*> ids;
    for (const auto& a : M->apps) ids.push_back(a.c_str());
    ocg_matrix* checked = nullptr;  // same validation as a matrix built from arrays
    int rc = ocg_matrix_create(m, n, ids.data(), M->cpu.data(), M->gpu.data(), M->rp.data(), M->col.data(),
                               M->val.data(), &checked);
    if (rc) return rc;
    *out = checked;
    return OCG_OK;
}

void ocg_matrix_destroy(ocg_matrix* M) { delete M; }

// ------------------------------------------------------------ predictor
int ocg_predictor_parse(const char* text, int32_t* n_layers, int64_t* dims, int32_t* acts, double* params,
                        int64_t* nparams, double* mean7, double* std7, int* has_stats) {
    if (!text) return fail(OCG_E_INVALID, "null argument");
    PredModel pm;
    int rc = parse_predictor(text, pm);
    if (rc) return rc;
    if (n_layers) *n_layers = static_cast<int32_t>(pm.acts.size());
    if (nparams) *nparams = static_cast<int64_t>(pm.params.size());
    if (dims) std::copy(pm.dims.begin(), pm.dims.end(), dims);
    if (acts) std::copy(pm.acts.begin(), pm.acts.end(), acts);
    if (params) std::copy(pm.params.begin(), pm.params.end(), params);
    if (mean7) std::copy(pm.mean, pm.mean + 7, mean7);
    if (std7) std::copy(pm.sd, pm.sd + 7, std7);
    if (has_stats) *has_stats = pm.has_stats ? 1 : 0;
    return OCG_OK;
}

int ocg_predictor_from_json(ocg_ctx* ctx, const char* text, ocg_predictor** out) {
    if (!ctx || !text || !out) return fail(OCG_E_INVALID, "null argument");
    PredModel pm;
    int rc = parse_predictor(text, pm);
    if (rc) return rc;
    return ocg_predictor_create(ctx, static_cast<int32_t>(pm.acts.size()), pm.dims.data(), pm.acts.data(),
                                pm.params.data(), pm.mean, pm.sd, pm.has_stats ? 1 : 0, out);
}

int ocg_predictor_load(ocg_ctx* ctx, const char* path, ocg_predictor** out) {
    if (!path) return fail(OCG_E_INVALID, "null argument");
    std::string text;
    int rc = read_file(path, text, "predictor model");  // predictor.cpp:327-328
    if (rc) return rc;
    return ocg_predictor_from_json(ctx, text.c_str(), out);
}

}  // extern "C"
