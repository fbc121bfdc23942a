// hgks_b200/io.hpp — the result tables and CSV writers of the reference's
// drivers (proj/include/hgks/io.hpp:17-21, :147-215), for numbers produced by
// the B200 path. The key=value run-config loader of io.hpp:23-145 belongs to
// the CLI and is out of scope. Output is byte-identical to the
// reference's writers ("%.17g").
#pragma once

#include <cmath>
#include <cstdio>
#include <optional>
#include <ostream>
#include <string>
#include <vector>

#include "hgks.hpp"

namespace hgks {

inline std::string fmt17(double v) {
    char b[64];
    std::snprintf(b, sizeof b, "%.17g", v);
    return b;
}

struct ErrorRow {
    int n;
    ErrorNorms e;
    std::optional<double> order_l1, order_l2, order_c;
};

/// orders log2(e_coarse / e_fine) between consecutive meshes, none on the first row
inline std::vector<ErrorRow> make_error_table(const std::vector<int>& meshes, const std::vector<ErrorNorms>& errs) {
    std::vector<ErrorRow> rows;
    for (size_t i = 0; i < meshes.size(); ++i) {
        ErrorRow r{meshes[i], errs[i], {}, {}, {}};
        if (i > 0) {
            r.order_l1 = std::log2(errs[i - 1].l1 / errs[i].l1);
            r.order_l2 = std::log2(errs[i - 1].l2 / errs[i].l2);
            r.order_c = std::log2(errs[i - 1].cell_avg / errs[i].cell_avg);
        }
        rows.push_back(r);
    }
    return rows;
}

inline void write_errors_csv(std::ostream& os, const std::vector<ErrorRow>& rows) {
    auto opt = [](const std::optional<double>& v) { return v ? fmt17(*v) : std::string(); };
    os << "mesh,eL1,orderL1,eL2,orderL2,ec,orderc\n";
    for (const auto& r : rows)
        os << r.n << ',' << fmt17(r.e.l1) << ',' << opt(r.order_l1) << ',' << fmt17(r.e.l2) << ','
           << opt(r.order_l2) << ',' << fmt17(r.e.cell_avg) << ',' << opt(r.order_c) << '\n';
}

inline void write_tgv_csv(std::ostream& os, const std::vector<TgvRecord>& recs) {
    os << "t,Ek,epsEk,epsZeta\n";
    for (const auto& r : recs)
        os << fmt17(r.t) << ',' << fmt17(r.Ek) << ',' << fmt17(r.epsEk) << ',' << fmt17(r.epsZeta) << '\n';
}

inline void write_scaling_csv(std::ostream& os, const std::vector<ScalingRow>& rows) {
    os << "size,workers,seconds,speedup\n";
    for (const auto& r : rows)
        os << r.size << ',' << r.workers << ',' << fmt17(r.seconds) << ',' << fmt17(r.speedup) << '\n';
}

/// cell-average primitive fields
inline void write_fields_csv(std::ostream& os, const RunResult& r, const GasModel& gas) {
    os << "i,j,k,x,y,z,rho,u,v,w,p\n";
    for (int c = 0; c < r.mesh.ncells(); ++c) {
        const auto ijk = r.mesh.cell_ijk(c);
        const auto x = r.mesh.center(c);
        const Conserved q{r.state.coeff(c, 0, 0), r.state.coeff(c, 0, 1), r.state.coeff(c, 0, 2),
                          r.state.coeff(c, 0, 3), r.state.coeff(c, 0, 4)};
        const Primitive w = primitive_from_conserved(q, gas);
        os << ijk[0] << ',' << ijk[1] << ',' << ijk[2] << ',' << fmt17(x[0]) << ',' << fmt17(x[1]) << ','
           << fmt17(x[2]) << ',' << fmt17(w.rho) << ',' << fmt17(w.U) << ',' << fmt17(w.V) << ',' << fmt17(w.W)
           << ',' << fmt17(pressure(w)) << '\n';
    }
}

inline void write_coeffs_csv(std::ostream& os, const RunResult& r) {
    os << "cell,n,rho,mx,my,mz,E\n";
    for (int c = 0; c < r.state.ncells; ++c)
        for (int n = 0; n < r.state.N; ++n) {
            os << c << ',' << n;
            for (int v = 0; v < 5; ++v) os << ',' << fmt17(r.state.coeff(c, n, v));
            os << '\n';
        }
}

}  // namespace hgks
