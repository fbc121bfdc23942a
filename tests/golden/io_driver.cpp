// Feeds fixed numbers through the REFERENCE's own CSV writers
// (proj/include/hgks/io.hpp) to produce the golden files tests/test_io.py
// compares the device-side writers (paper_2202_13821_b200/io.py) against.
// Built and run by make_io_golden.py in the build container only.
#include <cstdio>
#include <fstream>
#include <iostream>
#include <string>
#include <vector>

#include "hgks/io.hpp"
#include "hgks/solver.hpp"

int main(int argc, char** argv) {
    if (argc != 3) return 2;
    std::ifstream in(argv[1]);
    const std::string out = argv[2];
    int ne;
    in >> ne;
    std::vector<int> meshes(ne);
    std::vector<hgks::ErrorNorms> errs(ne);
    for (int i = 0; i < ne; ++i) in >> meshes[i] >> errs[i].l1 >> errs[i].l2 >> errs[i].cell_avg;
    int nt;
    in >> nt;
    std::vector<hgks::TgvRecord> recs(nt);
    for (auto& r : recs) in >> r.t >> r.Ek >> r.epsEk >> r.epsZeta;
    int ns;
    in >> ns;
    std::vector<hgks::ScalingRow> rows(ns);
    for (auto& r : rows) in >> r.size >> r.workers >> r.seconds >> r.speedup;
    int nx, ny, nz, N;
    double gamma;
    in >> nx >> ny >> nz >> N >> gamma;
    std::vector<double> xs(nx + 1), ys(ny + 1), zs(nz + 1);
    for (auto& v : xs) in >> v;
    for (auto& v : ys) in >> v;
    for (auto& v : zs) in >> v;
    hgks::RunResult r;
    r.mesh = hgks::Mesh::make(xs, ys, zs);
    r.state = hgks::DGState::zeros(r.mesh.ncells(), N);
    for (auto& v : r.state.coeffs) in >> v;
    if (!in) return 3;
    const hgks::GasModel gas = hgks::GasModel::make(gamma, 0.0);
    std::ofstream(out + "/errors.csv") << "";
    {
        std::ofstream f(out + "/errors.csv");
        hgks::write_errors_csv(f, hgks::make_error_table(meshes, errs));
    }
    {
        std::ofstream f(out + "/tgv.csv");
        hgks::write_tgv_csv(f, recs);
    }
    {
        std::ofstream f(out + "/scale.csv");
        hgks::write_scaling_csv(f, rows);
    }
    {
        std::ofstream f(out + "/fields.csv");
        hgks::write_fields_csv(f, r, gas);
    }
    {
        std::ofstream f(out + "/coeffs.csv");
        hgks::write_coeffs_csv(f, r);
    }
    return 0;
}
