/* kernelweave B200 drop-in — matrix CSV I/O (reference: core/include/kernelweave/buffer_csv.hpp,
 * core/src/buffer_csv.cpp; pinned by test_buffer.cpp:275-310).
 *
 * Same text format as the reference, byte for byte: one line per row, ',' between values, each
 * value printed "%.17g" (17 significant digits identify a double, so parse + print is the
 * identity on the text). Same errors: only 2-D double buffers are written; ragged, empty or
 * malformed input is a UsageError. In this build a buffer may live on a GPU: it is staged
 * through page-locked host memory with a synchronous queue on its device. */
#pragma once

#include "kernelweave/buffer.hpp"
#include "kernelweave/queue.hpp"

#include <cstdio>
#include <cstdlib>
#include <istream>
#include <optional>
#include <ostream>
#include <string>
#include <vector>

namespace kernelweave {

namespace detail {

/// The host image of a GPU buffer: a page-locked copy made through a synchronous queue.
inline Buffer hostCopy(const Buffer& buf)
{
    Buffer staging(Device::host(), buf.extent(), buf.elemSize());
    Queue q(buf.device(), QueueFlavor::Sync);
    copyBuffer(q, staging, buf, buf.extent());
    q.wait();
    return staging;
}

/// Splits one CSV line into doubles with strtod (the reference accepts what strtod accepts:
/// leading blanks, signs, exponents, inf/nan; a trailing '\r' ends the line).
inline std::vector<double> parseCsvLine(const std::string& line)
{
    std::vector<double> values;
    const char* p = line.c_str();
    while (true) {
        char* next = nullptr;
        const double v = std::strtod(p, &next);
        if (next == p)
            throw UsageError("readBufferCsv: malformed number in '" + line + "'");
        values.push_back(v);
        if (*next == ',') {
            p = next + 1;
            continue;
        }
        if (*next != '\0' && *next != '\r')
            throw UsageError("readBufferCsv: unexpected character in '" + line + "'");
        return values;
    }
}

} // namespace detail

/// Writes a 2-D double buffer as CSV (buffer_csv.hpp:14-16).
inline void writeBufferCsv(const Buffer& buf, std::ostream& os)
{
    if (buf.dim() != 2)
        throw UsageError("writeBufferCsv: only 2-D buffers are supported");
    if (buf.elemSize() != sizeof(double))
        throw UsageError("writeBufferCsv: only double elements are supported");
    std::optional<Buffer> staging;
    if (!buf.device().isHost())
        staging.emplace(detail::hostCopy(buf));
    const Buffer& img = staging ? *staging : buf;
    std::string line;
    char text[40];
    for (std::size_t r = 0; r < img.extent()[0]; ++r) {
        line.clear();
        const double* row = img.rowData<double>(r);
        for (std::size_t c = 0; c < img.extent()[1]; ++c) {
            std::snprintf(text, sizeof text, c ? ",%.17g" : "%.17g", row[c]);
            line += text;
        }
        line += '\n';
        os << line;
    }
}

/// Parses a CSV matrix into a new 2-D double buffer on `device` (buffer_csv.hpp:18-20).
inline Buffer readBufferCsv(std::istream& is, Device device = Device::host())
{
    std::vector<double> values;
    std::size_t rows = 0, cols = 0;
    std::string line;
    while (std::getline(is, line)) {
        if (line.empty() && is.eof())
            break; // a final newline, not an empty row
        const std::vector<double> row = detail::parseCsvLine(line);
        if (rows > 0 && row.size() != cols)
            throw UsageError("readBufferCsv: ragged rows");
        cols = row.size();
        values.insert(values.end(), row.begin(), row.end());
        ++rows;
    }
    if (rows == 0 || cols == 0)
        throw UsageError("readBufferCsv: empty input");
    Buffer host(Device::host(), IndexVec(rows, cols), sizeof(double));
    for (std::size_t r = 0; r < rows; ++r) {
        double* out = host.rowData<double>(r);
        for (std::size_t c = 0; c < cols; ++c)
            out[c] = values[r * cols + c];
    }
    if (device.isHost())
        return host;
    Buffer dev(device, host.extent(), sizeof(double));
    Queue q(device, QueueFlavor::Sync);
    copyBuffer(q, dev, host, host.extent());
    q.wait();
    return dev;
}

} // namespace kernelweave
