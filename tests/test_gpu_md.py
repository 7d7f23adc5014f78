"""Device-resident MD loop: nnmd_b200_run_md against the reference's
run_md arithmetic (engine.cpp:91-100 leapfrog_step, system.cpp:59-69 wrap_position,
engine.cpp:171-180 on-step kinetic energy, engine.cpp:132-141 rescaling), restated here in
numpy on the forces of the same CUDA path.  Given identical forces the integrator is
bit-identical, so positions, velocities and potential energies must match exactly; the
total energy differs only by the kinetic-energy summation order."""
import numpy as np
import pytest

import paper_2604_07276_b200 as nb

pytestmark = pytest.mark.gpu


def host_leapfrog(pos, vel, mass, f, dt, L):
    """leapfrog_step + wrap_position + run_md's mid-point kinetic energy, in FP64."""
    inv_m = 1.0 / mass
    v_old = vel.copy()
    vel += (dt * inv_m)[:, None] * f
    pos += dt * vel
    w = pos - np.floor(pos / L) * L
    w[w >= L] = 0.0
    pos[...] = w
    vm = 0.5 * (v_old + vel)
    return float(np.sum((0.5 * mass) * ((vm[:, 0] * vm[:, 0] + vm[:, 1] * vm[:, 1]) + vm[:, 2] * vm[:, 2])))


def rescale(vel, mass, temperature):
    ke = float(np.sum((0.5 * mass) * ((vel[:, 0] ** 2 + vel[:, 1] ** 2) + vel[:, 2] ** 2)))
    if ke > 0:
        vel *= np.sqrt(temperature / (2.0 * ke / (3.0 * len(vel))))


def system(n=300, seed=5):
    box, pos, sp = nb.synth_system(n, 0.1, 0.9, seed)
    rng = np.random.default_rng(seed)
    mass = np.where(sp == 0, 1.008, 12.0).astype(np.float64)
    vel = rng.normal(0.0, 0.05, size=(n, 3))
    vel -= (mass[:, None] * vel).sum(0) / mass.sum()
    return box, np.ascontiguousarray(pos), sp, mass, np.ascontiguousarray(vel)


@pytest.mark.parametrize("n_ranks", [1, 2])
def test_device_loop_matches_host_integrator_bitwise(n_ranks):
    box, pos, sp, mass, vel = system()
    m = nb.init_model(nb.test_spec(4.0, n_species=6), 5)
    ev = nb.DeviceEvaluator(m, n_ranks=n_ranks)
    steps, dt = 6, 0.0005
    hp, hv = pos.copy(), vel.copy()
    h_pot, h_tot = [], []
    for _ in range(steps):
        r = ev.compute(hp, sp, box)
        ke = host_leapfrog(hp, hv, mass, r["forces"], dt, box)
        h_pot.append(r["energy"])
        h_tot.append(r["energy"] + ke)
    dp, dv = pos.copy(), vel.copy()
    pot, tot = ev.run_md(dp, dv, mass, sp, box, dt, steps)
    assert np.array_equal(dp, hp)
    assert np.array_equal(dv, hv)
    assert np.array_equal(pot, np.array(h_pot))
    assert np.abs(tot - np.array(h_tot)).max() <= 1e-13 * np.abs(h_tot).max()


def test_device_loop_rescaling():
    box, pos, sp, mass, vel = system(seed=9)
    m = nb.init_model(nb.test_spec(4.0, n_species=6), 2)
    ev = nb.DeviceEvaluator(m, n_ranks=1)
    steps, dt, T = 6, 0.0005, 0.02
    hp, hv = pos.copy(), vel.copy()
    for k in range(steps):
        r = ev.compute(hp, sp, box)
        host_leapfrog(hp, hv, mass, r["forces"], dt, box)
        if k < 4 and (k + 1) % 2 == 0:
            rescale(hv, mass, T)
    dp, dv = pos.copy(), vel.copy()
    ev.run_md(dp, dv, mass, sp, box, dt, steps, equil_steps=4, target_temperature=T, rescale_every=2)
    # the kinetic-energy sum order differs (device tree vs numpy): last-bit differences only
    assert np.abs(dv - hv).max() <= 1e-12 * np.abs(hv).max()
    assert np.abs(dp - hp).max() <= 1e-12 * box.max()
    ke = 0.5 * np.sum(mass[:, None] * dv * dv)
    assert abs(2 * ke / (3 * len(dv)) - T) / T < 0.5  # rescaled towards T, then two free steps


def test_device_loop_energy_conservation_and_api():
    box, pos, sp, mass, vel = system(n=400, seed=3)
    m = nb.init_model(nb.test_spec(4.0, n_species=6), 4)
    prov = nb.DpProvider(m, nb.DpProvider.Options(decomposed=True, scheme=nb.MASKED_REDUCTION, n_ranks=2))
    atoms = nb.AtomSet(np.arange(len(pos), dtype=np.int64), sp, pos.copy(), vel.copy(), mass)
    s = nb.run_md(atoms, nb.SimBox(box), nb.MDConfig(dt=0.0002, n_steps=40), prov)
    assert s.steps == 40 and len(s.total_energy) == 40 and s.throughput > 0
    drift = np.abs(s.total_energy - s.total_energy[0]).max()
    assert drift <= 1e-3 * max(np.abs(s.potential_energy).max(), 1e-12)
    assert np.all((atoms.positions >= 0) & (atoms.positions < box))


def test_device_loop_non_finite_force_is_an_error():
    box, pos, sp, mass, vel = system(n=200, seed=4)
    pos[1] = pos[0]  # coincident atoms: r = 0 -> non-finite switch and forces
    m = nb.init_model(nb.test_spec(4.0, n_species=6), 4)
    ev = nb.DeviceEvaluator(m, n_ranks=1)
    with pytest.raises(nb.Error, match="non-finite force"):
        ev.run_md(pos, vel, mass, sp, box, 0.0005, 3)
