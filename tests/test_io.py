"""File formats (paper_2509_00774_b200.io) against files the REFERENCE wrote
(tests/golden/io/, made by tests/golden/make_io_golden.py) and the reference's own io test
strategy (pkg/tests/test_io.py): bit-exact round trips, corruption detection, fuzzing,
schema errors naming the key path, and CSV slices. CPU only."""

from __future__ import annotations

import json
import struct
from pathlib import Path

import numpy as np
import pytest

from conftest import small, tiny
from paper_2509_00774_b200 import (
    ArrayGeometry,
    ConstantPulse,
    FrequencyGrid,
    ImagingScenario,
    MeasurementSet,
    ReflectivityVolume,
    TabulatedPulse,
    Vec3,
    VoxelGrid,
    make_spiral_array,
    preset_scenario,
    scenario_fingerprint,
)
from paper_2509_00774_b200.io import (
    BadMagicError,
    ChecksumError,
    FingerprintMismatchError,
    FormatError,
    SchemaError,
    TruncatedFileError,
    VersionError,
    export_slices_csv,
    read_measurements,
    read_scenario,
    read_volume,
    write_measurements,
    write_scenario,
    write_volume,
)

GOLD = Path(__file__).resolve().parent / "golden" / "io"


@pytest.fixture(scope="module")
def inputs():
    return np.load(GOLD / "inputs.npz")


def golden_grid():
    return VoxelGrid(center=Vec3(0.01, -0.02, 0.4), extent=(0.1, 0.15, 0.05), dims=(3, 4, 2))


def golden_scenarios():
    tab = ImagingScenario(
        array=ArrayGeometry(transmitters=(Vec3(0.05, 0.0, 0.0), Vec3(-0.05, 0.02, 0.0)),
                            receivers=(Vec3(0.0, 0.04, 0.0),)),
        frequencies=FrequencyGrid(5e9, 7e9, 3),
        voxels=VoxelGrid(center=Vec3(0.0, 0.0, 0.35), extent=(0.1, 0.1, 0.0), dims=(2, 2, 1)),
        pulse=TabulatedPulse((4e9, 6e9, 8e9), (1 + 0j, 0.5 - 0.25j, 0.1 + 0.3j)),
    )
    return {"tabulated": tab, "small": small(), "paper_v": preset_scenario("paper-v")}


# ------------------------------------------------------------------ parity with the reference's files


def test_writers_match_reference_bytes(inputs, tmp_path):
    vol = ReflectivityVolume(inputs["volume"], golden_grid())
    write_volume(vol, tmp_path / "v.nfmv")
    assert (tmp_path / "v.nfmv").read_bytes() == (GOLD / "volume.nfmv").read_bytes()
    g1 = VoxelGrid(center=Vec3(0, 0, 0.3), extent=(0, 0, 0), dims=(1, 1, 1))
    write_volume(ReflectivityVolume(np.array([0.3 - 0.4j]), g1), tmp_path / "s.nfmv")
    assert (tmp_path / "s.nfmv").read_bytes() == (GOLD / "single.nfmv").read_bytes()
    write_measurements(MeasurementSet.for_scenario(inputs["measurements"], small()), tmp_path / "m.nfms")
    assert (tmp_path / "m.nfms").read_bytes() == (GOLD / "small.nfms").read_bytes()
    for name, scn in golden_scenarios().items():
        write_scenario(scn, tmp_path / f"{name}.json")
        assert (tmp_path / f"{name}.json").read_text() == (GOLD / f"{name}.json").read_text(), name
    paths = export_slices_csv(vol, tmp_path / "slices")
    assert [p.name for p in paths] == ["slices_z0.csv", "slices_z1.csv"]
    for p in paths:
        assert p.read_text() == (GOLD / p.name).read_text()


def test_readers_decode_reference_files(inputs):
    vol = read_volume(GOLD / "volume.nfmv", grid=golden_grid())
    assert np.array_equal(vol.values, inputs["volume"])
    m = read_measurements(GOLD / "small.nfms", scenario=small())
    assert np.array_equal(m.values, inputs["measurements"])
    for name, fp in zip(inputs["names"], inputs["fingerprints"]):
        scn = read_scenario(GOLD / f"{name}.json")
        assert scenario_fingerprint(scn) == bytes(fp.tolist()), name
        assert scn == golden_scenarios()[str(name)]


# ------------------------------------------------------------------ volumes / measurements


def test_volume_round_trip_and_unit_grid(tmp_path, rng):
    grid = golden_grid()
    vals = rng.standard_normal(grid.n_voxels) + 1j * rng.standard_normal(grid.n_voxels)
    p = tmp_path / "v.nfmv"
    write_volume(ReflectivityVolume(vals, grid), p)
    assert np.array_equal(read_volume(p, grid=grid).values, vals)
    unit = read_volume(p).grid
    assert unit.dims == (3, 4, 2) and unit.spacing == (1.0, 1.0, 1.0) and unit.center == Vec3(0, 0, 0)
    with pytest.raises(ValueError, match="dims"):
        read_volume(p, grid=VoxelGrid(center=Vec3(0, 0, 0), extent=(1, 1, 1), dims=(2, 4, 3)))


def test_volume_corruptions(tmp_path):
    blob = (GOLD / "volume.nfmv").read_bytes()
    p = tmp_path / "x.nfmv"
    cases = [
        (blob[:-1], TruncatedFileError),
        (blob[:10], TruncatedFileError),
        (blob + b"\0", TruncatedFileError),
        (b"NFMX" + blob[4:], BadMagicError),
        (blob[:4] + struct.pack("<H", 2) + blob[6:], VersionError),
        (blob[:40] + bytes([blob[40] ^ 0x10]) + blob[41:], ChecksumError),
        (blob[:-8] + struct.pack("<Q", 7), ChecksumError),
        (struct.pack("<4sHIII", b"NFMV", 1, 0, 4, 2) + blob[18:], SchemaError),
    ]
    for data, err in cases:
        p.write_bytes(data)
        with pytest.raises(err):
            read_volume(p)


def test_measurements_pairing_and_extra_bytes(tmp_path, rng):
    scn = small()
    p = tmp_path / "m.nfms"
    write_measurements(MeasurementSet.for_scenario(rng.standard_normal(scn.n_channels) + 0j, scn), p)
    assert read_measurements(p).fingerprint == scenario_fingerprint(scn)
    with pytest.raises(FingerprintMismatchError):
        read_measurements(p, scenario=tiny())
    p.write_bytes(p.read_bytes() + b"junk")
    with pytest.raises(TruncatedFileError):
        read_measurements(p)
    # a correct fingerprint with a different channel count
    q = tmp_path / "short.nfms"
    write_measurements(MeasurementSet(np.zeros(3, complex), scenario_fingerprint(scn)), q)
    with pytest.raises(FingerprintMismatchError, match="channels"):
        read_measurements(q, scenario=scn)


def test_fuzzed_files_raise_format_errors(tmp_path, rng):
    seeds = [((GOLD / "volume.nfmv").read_bytes(), read_volume),
             ((GOLD / "small.nfms").read_bytes(), lambda q: read_measurements(q, scenario=small()))]
    target = tmp_path / "fuzz.bin"
    for blob, reader in seeds:
        for _ in range(300):
            data = bytearray(blob)
            op = int(rng.integers(0, 3))
            if op == 0:
                data[int(rng.integers(0, len(data)))] ^= int(rng.integers(1, 256))
            elif op == 1:
                data = data[: int(rng.integers(0, len(data)))]
            else:
                data += bytes(rng.integers(0, 256, size=int(rng.integers(1, 64))).tolist())
            target.write_bytes(bytes(data))
            with pytest.raises(FormatError):
                reader(target)


def test_noise_and_huge_claims_rejected(tmp_path, rng):
    t = tmp_path / "noise.bin"
    t.write_bytes(bytes(rng.integers(0, 256, size=1_000_000, dtype=np.uint8)))
    for reader in (read_volume, read_measurements):
        with pytest.raises(FormatError):
            reader(t)
    h = tmp_path / "huge.nfmv"
    h.write_bytes(struct.pack("<4sHIII", b"NFMV", 1, 2**32 - 1, 2**32 - 1, 4) + b"\0" * 64)
    with pytest.raises(TruncatedFileError):
        read_volume(h)


# ------------------------------------------------------------------ scenario documents


def _doc(scn=None) -> dict:
    from paper_2509_00774_b200.geometry import scenario_to_document

    return scenario_to_document(scn or tiny())


@pytest.mark.parametrize("mutate,match", [
    (lambda d: d.pop("receivers"), "missing key receivers"),
    (lambda d: d["voxels"].update(spacing=[1, 1, 1]), "unknown key voxels.spacing"),
    (lambda d: d.update(extra=1), "unknown key extra"),
    (lambda d: d["frequencies"].update(count=0), "invalid scenario document"),
    (lambda d: d["frequencies"].update(count=2.0), "frequencies.count must be an integer"),
    (lambda d: d["frequencies"].update(start_hz=True), "frequencies.start_hz must be a number"),
    (lambda d: d["voxels"].update(dims=[2, 2]), "voxels.dims must be a list of 3 numbers"),
    (lambda d: d["voxels"].update(dims=[2, 2, 1.5]), "voxels.dims must contain integers"),
    (lambda d: d["voxels"].update(center=[0, "a", 0]), "voxels.center must contain numbers only"),
    (lambda d: d.update(transmitters=[]), "transmitters must be a non-empty list"),
    (lambda d: d.update(receivers=[[0, 0]]), r"receivers\[0\] must be an \[x, y, z\] triple"),
    (lambda d: d.update(pulse={"mode": "chirp"}), "pulse.mode must be"),
    (lambda d: d.update(pulse={"mode": "constant", "value": [1]}), r"pulse.value must be a \[re, im\] pair"),
    (lambda d: d.update(pulse={"mode": "constant", "value": [1, 0], "x": 1}), "unknown key pulse.x"),
    (lambda d: d.update(pulse=[1]), "pulse must be an object"),
    (lambda d: d.update(frequencies=[1]), "frequencies must be an object"),
    (lambda d: d.update(speed_of_light="c"), "speed_of_light must be a number"),
])
def test_schema_errors_name_the_key_path(tmp_path, mutate, match):
    d = _doc()
    mutate(d)
    p = tmp_path / "s.json"
    p.write_text(json.dumps(d))
    with pytest.raises(SchemaError, match=match):
        read_scenario(p)


def test_scenario_round_trips(tmp_path):
    for scn in [tiny(), small(), preset_scenario("paper-v"),
                ImagingScenario(array=make_spiral_array(5, 4, 0.2, rng_seed=1),
                                frequencies=FrequencyGrid(1e9, 2e9, 7),
                                voxels=VoxelGrid(center=Vec3(0.1, -0.2, 0.7), extent=(0.3, 0.1, 0.2), dims=(4, 3, 2)),
                                pulse=ConstantPulse(0.25 - 1.5j), c=3.1e8)]:
        p = tmp_path / "s.json"
        write_scenario(scn, p)
        back = read_scenario(p)
        assert back == scn and scenario_fingerprint(back) == scenario_fingerprint(scn)
    (tmp_path / "bad.json").write_text("{not json")
    with pytest.raises(SchemaError, match="not valid JSON"):
        read_scenario(tmp_path / "bad.json")
    (tmp_path / "list.json").write_text("[1, 2]")
    with pytest.raises(SchemaError, match="JSON object"):
        read_scenario(tmp_path / "list.json")


# ------------------------------------------------------------------ CSV slices


def test_slices_csv_edge_cases(tmp_path):
    g1 = VoxelGrid(center=Vec3(0, 0, 0.3), extent=(0, 0, 0), dims=(1, 1, 1))
    (p,) = export_slices_csv(ReflectivityVolume(np.array([0.3 - 0.4j]), g1), tmp_path / "one")
    assert p.read_text() == "1\n"
    g = VoxelGrid(center=Vec3(0, 0, 0.3), extent=(0.1, 0.1, 0.1), dims=(2, 3, 2))
    paths = export_slices_csv(ReflectivityVolume.zeros(g), tmp_path / "zero")
    assert len(paths) == 2 and all(q.read_text() == "0,0\n0,0\n0,0\n" for q in paths)
    vals = np.arange(1, 13, dtype=float) + 0j  # flat x-fastest order: row y of slice z holds n = x + 2(y + 3z)
    paths = export_slices_csv(ReflectivityVolume(vals, g), tmp_path / "ramp")
    rows = [list(map(float, line.split(","))) for line in paths[1].read_text().splitlines()]
    assert rows == [[7 / 12, 8 / 12], [9 / 12, 10 / 12], [11 / 12, 1.0]]
