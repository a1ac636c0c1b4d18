// MATPOWER text output of solved stages: the host half
// of the reference's matpower.format_case / write_case (matpower.py:146-190).
// Each value is printed with "%.10g" (matpower.py:146-148); glibc's printf and
// CPython's %-formatting are both correctly rounded, so the text is
// byte-identical; NaN prints as "nan" whatever its sign bit (CPython's rule).
#pragma once
#include <cmath>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <string>

namespace acopf {

inline void fmt_g10(double v, std::string& out) {
    char buf[40];
    int n;
    if (std::isnan(v)) n = snprintf(buf, sizeof buf, "nan");
    else n = snprintf(buf, sizeof buf, "%.10g", v);
    out.append(buf, (size_t)n);
}

// "mpc.<section> = [\n" + per row "\t" + values joined by "\t" + ";\n" + "];"
// (matpower.py:151-157: the section lines joined by "\n")
inline void fmt_matrix(const char* section, int64_t rows, const int64_t* row_ptr, const double* values,
                       std::string& out) {
    out += "mpc.";
    out += section;
    out += " = [";
    for (int64_t r = 0; r < rows; ++r) {
        out += "\n\t";
        for (int64_t k = row_ptr[r]; k < row_ptr[r + 1]; ++k) {
            if (k > row_ptr[r]) out += '\t';
            fmt_g10(values[k], out);
        }
        out += ';';
    }
    out += "\n];";
}

}  // namespace acopf
