// test_dropin.cpp -- the reference's hot-path doctest cases (tests/test_variational.cpp,
// tests/test_circuit.cpp, tests/test_hamiltonian.cpp), ported one-for-one onto the
// drop-in headers and run on the GPU.  A tiny CHECK harness stands in for doctest
// (not available offline).  Exit code = number of failed checks.
#include <cmath>
#include <cstdio>
#include <functional>
#include <string>
#include <vector>

#include "qforge/circuit.hpp"
#include "qforge/lattice.hpp"
#include "qforge/noise.hpp"
#include "qforge/shadows.hpp"
#include "qforge/variational.hpp"

using namespace qforge;

static int g_fail = 0, g_pass = 0;
static std::string g_case;
#define CHECK(cond)                                                                                   \
    do {                                                                                              \
        if (cond) ++g_pass;                                                                           \
        else { ++g_fail; std::printf("FAIL [%s] %s:%d: %s\n", g_case.c_str(), __FILE__, __LINE__, #cond); } \
    } while (0)
#define CHECK_THROWS(expr)                               \
    do {                                                 \
        bool threw_ = false;                             \
        try { (void)(expr); } catch (const std::invalid_argument&) { threw_ = true; } \
        CHECK(threw_);                                   \
    } while (0)
#define CHECK_NOTHROW(expr)                              \
    do {                                                 \
        bool ok_ = true;                                 \
        try { (void)(expr); } catch (...) { ok_ = false; } \
        CHECK(ok_);                                      \
    } while (0)
static bool approx(double a, double b, double eps) { return std::abs(a - b) <= eps * std::max(1.0, std::abs(b)); }
static void test_case(const char* name, const std::function<void()>& f) {
    g_case = name;
    try { f(); } catch (const std::exception& e) { ++g_fail; std::printf("FAIL [%s] exception: %s\n", name, e.what()); }
}

static PauliSum tfim_chain(int n, double g) { return tfim_terms(build_lattice(LatticeKind::chain, {n}, {false}), g); }
static AnsatzSpec single_rx() {
    AnsatzSpec a;
    a.n_params = 1;
    a.builder = [](const RealVector& t) { Circuit c(1); c.rx(0, t[0]); return c; };
    a.shift_eligible = {true};
    return a;
}

int main() {
    test_case("chain ansatz layout", [] {  // test_variational.cpp:33-53
        AnsatzSpec a = tfim_chain_ansatz(4, 3);
        a.validate();
        CHECK(a.n_params == 3 * (2 * 4 - 1));
        RealVector zero = RealVector::Zero(a.n_params);
        CHECK(approx(energy(a, zero, tfim_chain(4, 1.0)), -4.0, 1e-10));
        Circuit c = a.builder(zero);
        int h = 0, rx = 0, rzz = 0;
        for (const auto& op : c.ops) { h += op.name == Gate::h; rx += op.name == Gate::rx; rzz += op.name == Gate::rzz; }
        CHECK(h == 4 && rx == 12 && rzz == 9);
    });
    test_case("energy evaluation", [] {  // test_variational.cpp:55-101
        AnsatzSpec a;
        a.n_params = 0;
        a.builder = [](const RealVector&) { return Circuit(2); };
        CHECK(approx(energy(a, RealVector(), tfim_chain(2, 1.0)), -1.0, 1e-10));
        AnsatzSpec t = tfim_chain_ansatz(5, 2);
        RngStream rng(3);
        RealVector theta(t.n_params);
        for (int i = 0; i < t.n_params; ++i) theta[i] = rng.normal();
        PauliSum h = tfim_chain(5, 1.3);
        CHECK(energy(t, theta, h) == energy(t, theta, h));
        const double e1 = energy(t, theta, h), e3 = energy(t, theta, pauli_sum_to_coo(h));  // operator formats
        CHECK(approx(e1, e3, 1e-12));
    });
    test_case("shadow snapshots", [] {  // test_shadows.cpp:101-145, 184-193
        RngStream r1(1);
        auto ds = shadow_snapshots(StateVector::zero_state(3), std::vector<std::vector<int>>(50, {3, 3, 3}), r1);
        bool zeros = true;
        for (const auto& row : ds.outcomes)
            for (int b : row) zeros = zeros && b == 0;
        CHECK(zeros);
        Circuit plus(3);
        plus.h(0).h(1).h(2);
        RngStream r2(2);
        ds = shadow_snapshots(run(plus), std::vector<std::vector<int>>(50, {1, 1, 1}), r2);
        zeros = true;
        for (const auto& row : ds.outcomes)
            for (int b : row) zeros = zeros && b == 0;
        CHECK(zeros);
        RngStream r3(3);
        ds = shadow_snapshots(StateVector::zero_state(1), std::vector<std::vector<int>>(10000, {1}), r3);
        int ones = 0;
        for (const auto& row : ds.outcomes) ones += row[0];
        CHECK(std::abs(ones / 10000.0 - 0.5) < 3.0 * std::sqrt(0.25 / 10000.0));
        Circuit c(4);
        c.h(0).cx(0, 1).ry(2, 0.8).cx(2, 3);
        RngStream brng(7), a(9), b(9);
        auto bases = random_bases(64, 4, brng);
        CHECK(shadow_snapshots(run(c), bases, a, 1).outcomes == shadow_snapshots(run(c), bases, b, 4).outcomes);
        bool threw = false;
        try {
            RngStream r4(4);
            shadow_snapshots(StateVector::zero_state(1), {{0}}, r4);
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
        Circuit bell(2);
        bell.h(0).cx(0, 1);
        RngStream r5(21);
        auto bb = random_bases(10000, 2, r5);
        auto bds = shadow_snapshots(run(bell), bb, r5);
        CHECK(std::abs(estimate_pauli(bds, {1, 1}, 10) - 1.0) < 0.5);
        save_dataset(bds, "/tmp/qf_dropin_shadows.csv");
        auto back = load_dataset("/tmp/qf_dropin_shadows.csv");
        CHECK(back.bases == bds.bases && back.outcomes == bds.outcomes);
    });
    test_case("noise trajectories", [] {  // test_noise.cpp:175-195
        Circuit c(4);
        for (int q = 0; q < 4; ++q) c.h(q).rx(q, 0.3 + q);
        c.cx(0, 1).cx(1, 2).cx(2, 3);
        RngStream rng(3);
        Trajectory t = mc_trajectory(c, {}, rng);
        CHECK((t.state.amps - run(c).amps).cwiseAbs().maxCoeff() < 1e-12);
        CHECK(t.log_prob == 0.0);
        NoiseConf conf;
        conf.attach("x", amplitude_damping_channel(1.0));
        Circuit one(1);
        one.x(0);
        RngStream r5(5);
        for (const Trajectory& tr : mc_trajectories(one, conf, r5, 20)) {
            CHECK(approx(std::abs(tr.state.amps[0]), 1.0, 1e-12));
            CHECK(approx(tr.log_prob, 0.0, 1e-12));
        }
        CHECK(depolarizing_channel(0.05, 2).operators.size() == 16);
        CHECK(thermal_relaxation_channel(0.1, 0.2).completeness_defect() < 1e-12);
        NoiseConf wires;
        wires.attach_on_wires("cx", {1, 2}, depolarizing_channel(0.1, 2));
        int matched = 0;
        for (const auto& op : c.ops) matched += (int)wires.match(op).size();
        CHECK(matched == 1);
    });
    test_case("sparse operator", [] {  // pauli.cpp:89-153, sparse.cpp:44-51
        PauliSum h = tfim_chain(4, 0.7);
        SparseCOO m = pauli_sum_to_coo(h);
        CHECK(m.dim == 16 && m.nnz() == 16 * 5);
        for (size_t k = 1; k < m.nnz(); ++k)
            CHECK(m.rows[k - 1] < m.rows[k] || (m.rows[k - 1] == m.rows[k] && m.cols[k - 1] < m.cols[k]));
        SparseCOO twice = m + m;
        CHECK(twice.nnz() == m.nnz());
        ComplexVector v = ComplexVector::Zero(16);
        v[5] = 1.0;
        ComplexVector w = m.apply(v);
        CHECK(approx(w[5].real(), -1.0 * ((5 & 1) == ((5 >> 1) & 1) ? 1 : -1) - ((5 >> 1 & 1) == (5 >> 2 & 1) ? 1 : -1) -
                                      ((5 >> 2 & 1) == (5 >> 3 & 1) ? 1 : -1), 1e-12));
        bool threw = false;
        try {
            pauli_sum_to_coo(tfim_chain(27, 1.0));
        } catch (const std::invalid_argument&) {
            threw = true;
        }
        CHECK(threw);
    });
    test_case("gradients", [] {  // test_variational.cpp:103-154
        PauliSum z;
        z.n = 1;
        z.add(1.0, {3});
        RealVector theta(1);
        theta << M_PI / 3.0;
        for (GradMode m : {GradMode::parameter_shift, GradMode::adjoint}) {
            RealVector g = gradient(single_rx(), theta, z, m);
            CHECK(approx(g[0], -std::sin(M_PI / 3.0), 1e-10));
            RealVector gfd = gradient(single_rx(), theta, z, GradMode::finite_diff);
            CHECK(approx(gfd[0], g[0], 1e-6));
        }
        RealVector pi(1);
        pi << M_PI;
        CHECK(std::abs(gradient(single_rx(), pi, z, GradMode::parameter_shift)[0]) < 1e-8);
        AnsatzSpec a = tfim_chain_ansatz(6, 2);
        PauliSum h = tfim_chain(6, 0.8);
        RngStream rng(5);
        RealVector th(a.n_params);
        for (int i = 0; i < a.n_params; ++i) th[i] = rng.normal();
        RealVector gs = gradient(a, th, h, GradMode::parameter_shift);
        RealVector gf = gradient(a, th, h, GradMode::finite_diff);
        RealVector ga = gradient(a, th, h, GradMode::adjoint);
        CHECK((gs - gf).cwiseAbs().maxCoeff() < 1e-6);
        CHECK((gs - ga).cwiseAbs().maxCoeff() < 1e-11);
        CHECK((gs - gradient(a, th, h, GradMode::parameter_shift, 1e-5, 4)).cwiseAbs().maxCoeff() == 0.0);
        AnsatzSpec su;
        su.n_params = 1;
        su.builder = [](const RealVector& t) { Circuit c(2); c.su4(0, 1, std::vector<double>(15, 0.2)); c.rx(0, t[0]); return c; };
        su.shift_eligible = {false};
        CHECK_THROWS(gradient(su, RealVector::Zero(1), tfim_chain(2, 1.0), GradMode::parameter_shift));
        CHECK_NOTHROW(gradient(su, RealVector::Zero(1), tfim_chain(2, 1.0), GradMode::finite_diff));
    });
    test_case("adam updates", [] {  // test_variational.cpp:156-190
        AdamState st;
        RealVector theta = RealVector::Zero(2), grad(2);
        grad << 0.3, -7.0;
        adam_step(st, theta, grad, 0.05);
        CHECK(approx(theta[0], -0.05, 1e-6) && approx(theta[1], 0.05, 1e-6));
    });
    test_case("vqe driver", [] {  // test_variational.cpp:193-233
        AnsatzSpec a = tfim_chain_ansatz(2, 2);
        PauliSum h = tfim_chain(2, 1.0);
        RngStream rng(7);
        std::vector<RealVector> batch;
        for (int s = 0; s < 8; ++s) {
            RealVector t(a.n_params);
            for (int i = 0; i < a.n_params; ++i) t[i] = 0.1 * rng.normal();
            batch.push_back(t);
        }
        VqeResult r = vqe_run(a, batch, h, 300, 0.02, GradMode::parameter_shift);
        CHECK(approx(r.best_energy, -std::sqrt(5.0), 1e-3));
        CHECK(r.best_index >= 0 && r.traces.size() == 8);
        CHECK(r.traces[r.best_index].back() == r.best_energy);
        AnsatzSpec a3 = tfim_chain_ansatz(3, 1);
        RealVector t0 = RealVector::Constant(a3.n_params, 0.3);
        VqeResult r1 = vqe_run(a3, {t0}, tfim_chain(3, 1.0), 1, 0.0, GradMode::parameter_shift);
        CHECK(approx(r1.best_energy, energy(a3, t0, tfim_chain(3, 1.0)), 1e-12));
    });
    test_case("basic gate application", [] {  // test_circuit.cpp:37-80
        StateVector psi = run(Circuit(1).h(0));
        CHECK(std::abs(psi.amps[0] - 1.0 / std::sqrt(2.0)) < 1e-12);
        StateVector bell = run(Circuit(2).h(0).cx(0, 1));
        PauliSum zz, xx;
        zz.n = xx.n = 2;
        zz.add(1.0, {3, 3});
        xx.add(1.0, {1, 1});
        CHECK(approx(expectation_pauli(bell, zz).real(), 1.0, 1e-12));
        CHECK(approx(expectation_pauli(bell, xx).real(), 1.0, 1e-12));
        StateVector rx = run(Circuit(1).rx(0, M_PI));
        CHECK(std::abs(rx.amps[0]) < 1e-12 && std::abs(rx.amps[1] - cplx(0, -1)) < 1e-12);
        CHECK_THROWS(run(Circuit(30)));
        CHECK_THROWS(Circuit(2).cx(1, 1));
        CHECK_THROWS(Circuit(2).rx(2, 0.1));
        CHECK_THROWS(Circuit(2).rx(0, NAN));
    });
    test_case("pauli expectations", [] {  // test_circuit.cpp:83-118
        StateVector psi = StateVector::zero_state(1);
        PauliSum z;
        z.n = 1;
        z.add(1.0, {3});
        CHECK(approx(expectation_pauli(psi, z).real(), 1.0, 1e-12));
    });
    test_case("builder without a fixed template (per-theta path)", [] {
        // structure depends on theta: energies and shift gradients still evaluate
        // (per parameter set, on the device); the adjoint gradient needs the template
        AnsatzSpec a;
        a.n_params = 2;
        a.shift_eligible = {true, true};
        a.builder = [](const RealVector& th) {
            Circuit c(2);
            c.ry(0, th[0]);
            if (th[0] > 0) c.rx(1, th[1]);
            else c.ry(1, th[1]);
            c.cx(0, 1);
            return c;
        };
        PauliSum zz;
        zz.n = 2;
        zz.add(1.0, {3, 3});
        RealVector t = RealVector::Zero(2);
        t[0] = 0.4;
        t[1] = -0.3;
        // ry(0.4) x rx(-0.3) then cx: <Z0 Z1> = <Z1> before cx = cos(-0.3)
        CHECK(approx(energy(a, t, zz), std::cos(-0.3), 1e-12));
        RealVector g = gradient(a, t, zz, GradMode::parameter_shift);
        CHECK(approx(g[0], 0.0, 1e-12) && approx(g[1], -std::sin(-0.3), 1e-12));
        CHECK_THROWS(gradient(a, t, zz, GradMode::adjoint));
    });
    test_case("apply_local_unitary on three wires", [] {  // circuit.cpp:147-175 (generic k)
        // X (x) X (x) X on wires {2, 0, 1} maps |000> to |111>; a permutation
        // unitary on wires {0, 2, 1} checks the local-bit order (wires[0] most significant)
        StateVector psi = StateVector::zero_state(3);
        ComplexMatrix x3 = ComplexMatrix::Zero(8, 8);
        for (int i = 0; i < 8; ++i) x3(7 - i, i) = 1.0;
        apply_local_unitary(psi, x3, {2, 0, 1});
        CHECK(std::abs(psi.amps[7] - 1.0) < 1e-12);
        StateVector e = StateVector::zero_state(3);
        e.amps[0] = 0.0;
        e.amps[1] = 1.0;  // |001>: qubit 2 set
        ComplexMatrix shift = ComplexMatrix::Zero(8, 8);
        for (int i = 0; i < 8; ++i) shift((i + 1) % 8, i) = 1.0;  // local index l -> l + 1
        apply_local_unitary(e, shift, {0, 2, 1});  // local index of |001> = (q0, q2, q1) = 010 = 2 -> 3 = 011
        CHECK(std::abs(e.amps[3] - 1.0) < 1e-12);  // (q0, q2, q1) = (0, 1, 1) -> q1 = q2 = 1 = |011>
        CHECK_THROWS(apply_local_unitary(e, shift, {0, 0, 1}));
    });
    test_case("rzz lowering", [] {  // test_circuit.cpp:302-314
        StateVector a = run(Circuit(2).h(0).h(1).rzz(0, 1, 0.9));
        StateVector b = run(Circuit(2).h(0).h(1).cx(0, 1).rz(1, 0.9).cx(0, 1));
        cplx ratio = b.amps[0] / a.amps[0];
        CHECK((a.amps * ratio - b.amps).cwiseAbs().maxCoeff() < 1e-12);
    });
    test_case("spin model builders", [] {  // test_hamiltonian.cpp:115-148
        PauliSum h = tfim_terms(build_lattice(LatticeKind::chain, {3}, {false}), 0.7);
        CHECK(h.terms.size() == 5);
        CHECK(heisenberg_terms(build_lattice(LatticeKind::chain, {2}, {false}), 1, 1, 1).terms.size() == 3);
        CHECK(tfim_terms(build_lattice(LatticeKind::chain, {10}, {false}), 1.0).terms.size() == 19);
    });
    test_case("complex64 device precision", [] {
        set_device_precision(Precision::c64);
        AnsatzSpec a = hea_ansatz(10, 2);
        RealVector th(a.n_params);
        for (int i = 0; i < a.n_params; ++i) th[i] = std::sin(0.37 * i);
        PauliSum h = tfim_chain(10, 1.0);
        RealVector g64 = gradient(a, th, h, GradMode::adjoint);
        set_device_precision(Precision::c128);
        RealVector g128 = gradient(a, th, h, GradMode::adjoint);
        CHECK((g64 - g128).cwiseAbs().maxCoeff() <= 1e-5 * g128.cwiseAbs().maxCoeff());
    });
    std::printf("%d passed, %d failed\n", g_pass, g_fail);
    return g_fail;
}
