"""Host-side rows of SURVEY.md §8f: scene files (PLY/JSON), image writers and
the CLI harness, checked against fixtures produced by the real reference
(tests/golden/make_io_golden.py).  CPU except the CLI render paths (gpu)."""

from __future__ import annotations

import csv
import hashlib
import json

import numpy as np
import pytest

from conftest import GOLDEN


def _sha(path) -> str:
    return hashlib.sha256(path.read_bytes()).hexdigest()


@pytest.fixture(scope="module")
def io_golden():
    with np.load(GOLDEN / "io_golden.npz") as z:
        return {k: z[k] for k in z.files}


def test_load_ply_bitexact_vs_reference(io_golden):
    import paper_2409_08669_b200 as ab

    arrays, deg = ab.load_ply_arrays(GOLDEN / "io_scene_sh3.ply")
    assert deg == int(io_golden["ply_sh_degree"]) == 3
    for f in ("centers", "scales", "rotations", "opacities", "sh"):
        assert np.array_equal(getattr(arrays, f).view(np.uint64), io_golden[f"ply_{f}"].view(np.uint64)), f
    scene = ab.load_ply(GOLDEN / "io_scene_sh3.ply")
    assert len(scene) == 40 and scene.sh_degree == 3
    assert np.array_equal(scene.as_arrays().sh, io_golden["ply_sh"])


def test_save_ply_and_json_byte_identical(io_golden, tmp_path):
    import paper_2409_08669_b200 as ab

    orig = ab.SceneArrays(*(io_golden[f"orig_{f}"] for f in ("centers", "scales", "rotations", "opacities", "sh")))
    ab.save_ply(orig, tmp_path / "o.ply", sh_degree=3)
    assert _sha(tmp_path / "o.ply") == str(io_golden["ply_sha"]) == _sha(GOLDEN / "io_scene_sh3.ply")
    scene = ab.load_ply(GOLDEN / "io_scene_sh3.ply")
    ab.save_ply(scene, tmp_path / "a.ply")      # the reference's load -> save
    assert _sha(tmp_path / "a.ply") == str(io_golden["resave_sha"])
    arrays, deg = ab.load_ply_arrays(GOLDEN / "io_scene_sh3.ply")
    ab.save_ply(arrays, tmp_path / "b.ply", sh_degree=deg)
    assert _sha(tmp_path / "b.ply") == str(io_golden["resave_sha"])
    syn = ab.generate_synthetic(9, 25, ab.SyntheticSpec())
    ab.save_scene(syn, tmp_path / "g.json")
    ab.save_scene(syn, tmp_path / "g.ply")
    assert _sha(tmp_path / "g.json") == str(io_golden["gen_json_sha"])
    assert _sha(tmp_path / "g.ply") == str(io_golden["gen_ply_sha"])
    back = ab.load_json(tmp_path / "g.json").as_arrays()
    assert np.array_equal(back.centers, syn.as_arrays().centers)


def test_scene_file_errors_match_reference(tmp_path):
    import paper_2409_08669_b200 as ab

    (tmp_path / "x.txt").write_text("nope")
    with pytest.raises(ab.SceneFormatError):
        ab.load_scene(tmp_path / "x.txt")
    (tmp_path / "bad.ply").write_bytes(b"ply\nformat ascii 1.0\nend_header\n")
    with pytest.raises(ab.SceneFormatError, match="binary_little_endian"):
        ab.load_ply(tmp_path / "bad.ply")
    (tmp_path / "bad.json").write_text("{")
    with pytest.raises(ab.SceneFormatError, match="invalid JSON"):
        ab.load_json(tmp_path / "bad.json")
    (tmp_path / "z.json").write_text(json.dumps({"sh_degree": 0, "gaussians": [
        {"center": [0, 0, 0], "scale": [1, 1, 1], "rotation": [0, 0, 0, 0], "opacity": 0.5, "sh": [[0, 0, 0]]}]}))
    with pytest.raises(ab.SceneValidationError):
        ab.load_json(tmp_path / "z.json")
    # a non-finite raw value in a PLY element
    arrays, deg = ab.load_ply_arrays(GOLDEN / "io_scene_sh3.ply")
    blob = bytearray((GOLDEN / "io_scene_sh3.ply").read_bytes())
    end = blob.find(b"end_header\n") + len(b"end_header\n")
    blob[end:end + 4] = np.array([np.nan], dtype="<f4").tobytes()
    (tmp_path / "nan.ply").write_bytes(bytes(blob))
    with pytest.raises(ab.SceneValidationError, match="element 0"):
        ab.load_ply(tmp_path / "nan.ply")


def test_validate_scene_diagnostics():
    import paper_2409_08669_b200 as ab

    good = ab.generate_synthetic(3, 5)
    assert ab.validate_scene(good) == []
    g = good.gaussians[2]
    g.opacity = 1.5
    g.scale = np.array([0.1, -1.0, 0.1])
    diags = ab.validate_scene(good)
    assert {(d.index, d.field) for d in diags} == {(2, "opacity"), (2, "scale")}


def test_image_writers_byte_identical(io_golden, tmp_path):
    import paper_2409_08669_b200 as ab
    from paper_2409_08669_b200 import imageio as io

    pix = io_golden["img_pixels"]
    img = ab.Image(width=17, height=13, pixels=pix)
    lm = ab.LoadMap(width=17, height=13, counts=io_golden["load_counts"])
    io.write_png(img, tmp_path / "i.png")
    io.write_ppm(img, tmp_path / "i.ppm")
    io.write_pgm16(lm, tmp_path / "l.pgm")
    io.write_loadmap_png(lm, tmp_path / "l.png")
    assert _sha(tmp_path / "i.png") == str(io_golden["png_sha"])
    assert _sha(tmp_path / "i.ppm") == str(io_golden["ppm_sha"])
    assert _sha(tmp_path / "l.pgm") == str(io_golden["pgm_sha"])
    assert _sha(tmp_path / "l.png") == str(io_golden["loadpng_sha"])


def test_cli_camera_and_gen_scene(io_golden, tmp_path, capsys):
    from paper_2409_08669_b200 import cli

    (tmp_path / "cam.json").write_text(str(io_golden["cam_doc"]))
    cam = cli.load_camera(tmp_path / "cam.json")
    assert np.array_equal(cam.view_matrix, io_golden["cam_view_matrix"]) and cam.fx == float(io_golden["cam_fx"])
    rc = cli.main(["gen-scene", "--seed", "9", "--count", "25", "--output", str(tmp_path / "g.json")])
    assert rc == 0 and _sha(tmp_path / "g.json") == str(io_golden["gen_json_sha"])
    assert "wrote 25 gaussians (seed 9)" in capsys.readouterr().out
    # exit codes: 2 for input errors (sb/cli.py:343-353)
    assert cli.main(["render", str(tmp_path / "missing.ply"), "--camera", str(tmp_path / "cam.json"),
                     "--output", str(tmp_path / "o.png")]) == 2
    (tmp_path / "badcam.json").write_text('{"position": [0, 0, -3]}')
    assert cli.main(["bench", str(tmp_path / "g.json"), "--camera", str(tmp_path / "badcam.json")]) == 2
    with pytest.raises(SystemExit):
        cli.main(["render"])
    assert cli.BENCH_COLUMNS[0] == "scene" and len(cli.BENCH_COLUMNS) == 16


@pytest.mark.gpu
def test_cli_render_compare_loadmap_bench_on_gpu(tmp_path, oracle):
    """The harness end to end on the B200 path: image bytes equal the
    oracle's image written by the same writer, CSV schemas, monotone pairs."""
    import paper_2409_08669_b200 as ab
    from paper_2409_08669_b200 import cli
    from paper_2409_08669_b200 import imageio as io

    assert cli.main(["gen-scene", "--seed", "4", "--count", "3000", "--output", str(tmp_path / "s.ply")]) == 0
    cam_doc = {"position": [0.2, 0.1, -3.0], "target": [0, 0, 0], "fov_y_deg": 60, "width": 160,
               "height": 120, "background": [0.1, 0.2, 0.3]}
    (tmp_path / "cam.json").write_text(json.dumps(cam_doc))
    csvp = tmp_path / "b.csv"
    assert cli.main(["render", str(tmp_path / "s.ply"), "--camera", str(tmp_path / "cam.json"),
                     "--output", str(tmp_path / "o.png"), "--loadmap", str(tmp_path / "l.png"),
                     "--csv", str(csvp)]) == 0
    arrays, deg = ab.load_ply_arrays(tmp_path / "s.ply")
    cam = cli.load_camera(tmp_path / "cam.json")
    ref = oracle.run_pipeline(dict(centers=arrays.centers, scales=arrays.scales, rotations=arrays.rotations,
                                   opacities=arrays.opacities, sh=arrays.sh, sh_degree=deg), cam, "aabb")
    io.write_png(ab.Image(160, 120, ref["pixels"]), tmp_path / "ref.png")
    assert _sha(tmp_path / "o.png") == _sha(tmp_path / "ref.png")
    assert cli.main(["compare", str(tmp_path / "s.ply"), "--camera", str(tmp_path / "cam.json"),
                     "--csv", str(tmp_path / "c.csv"), "--no-figure"]) == 0
    rows = list(csv.DictReader(open(tmp_path / "c.csv")))
    assert [r["mode"] for r in rows] == ["baseline", "circle", "aabb"]
    assert len({r["image_sha256"] for r in rows}) == 1 and rows[0]["psnr_vs_first"] == "999.0"
    assert cli.main(["loadmap", str(tmp_path / "s.ply"), "--camera", str(tmp_path / "cam.json"),
                     "--output", str(tmp_path / "lm.png"), "--pgm", str(tmp_path / "lm.pgm")]) == 0
    assert cli.main(["bench", str(tmp_path / "s.ply"), "--camera", str(tmp_path / "cam.json"),
                     "--repetitions", "3", "--csv", str(csvp), "--no-figure"]) == 0
    rows = list(csv.DictReader(open(csvp)))
    assert list(rows[0].keys()) == cli.BENCH_COLUMNS and len(rows) == 2
    assert int(rows[1]["pairs"]) == len(ref["keys"]) and float(rows[1]["fps"]) > 0


@pytest.mark.parametrize("name", ["sh3_extreme", "sh0_shuffled", "sh1_small", "sh2_reversed"])
def test_ply_cases_host_path_matches_reference_digests(name, tmp_path):
    """The deterministic checkpoints of tests/ply_cases.py (extreme logits and
    log-scales across the exp / expit special-case thresholds, shuffled and
    extra properties) load to the same arrays as the real splatbench's
    load_ply (tests/golden/ply_digests.json); the device ingest is checked
    against the same digests in tests/test_gpu_ply.py."""
    import json

    import paper_2409_08669_b200 as ab
    from ply_cases import write_case

    want = json.loads((GOLDEN / "ply_digests.json").read_text())[name]
    path = write_case(tmp_path, name)
    assert hashlib.sha256(path.read_bytes()).hexdigest() == want["file_sha256"]
    with np.errstate(over="ignore"):
        arrays, _ = ab.load_ply_arrays(path)
    for f in ("centers", "scales", "rotations", "opacities", "sh"):
        got = hashlib.sha256(np.ascontiguousarray(getattr(arrays, f), dtype=np.float64).tobytes()).hexdigest()
        assert got == want[f], f


def test_ply_device_columns_follow_the_reference_layout():
    """adr_ply_activate's column map: x y z, scale, rot, opacity, then SH in
    (k, channel) order with f_rest channel-major (sb/scene.py:380-384)."""
    from paper_2409_08669_b200.scene_io import PlySchema

    schema = PlySchema(2)
    names = list(schema.names)[::-1]
    index = {nm: i for i, nm in enumerate(names)}
    cols = schema.device_columns(index)
    assert cols.dtype == np.int32 and cols.size == 11 + 3 * 9
    named = [names[c] for c in cols]
    assert named[:11] == ["x", "y", "z", "scale_0", "scale_1", "scale_2", "rot_0", "rot_1", "rot_2", "rot_3",
                          "opacity"]
    assert named[11:14] == ["f_dc_0", "f_dc_1", "f_dc_2"]
    assert named[14:17] == ["f_rest_0", "f_rest_8", "f_rest_16"]   # k = 1: channel c at c * (K - 1)
    assert named[-3:] == ["f_rest_7", "f_rest_15", "f_rest_23"]


def test_ply_source_memory_maps_large_files(tmp_path):
    """load_ply_device's host side: a large file is memory-mapped (header from
    a 1 MB probe, same body offset as the whole blob), and a header whose
    end marker lies beyond the probe is still found (the reference searches
    the whole file, sb/scene.py:327)."""
    from paper_2409_08669_b200.scene_io import _HEADER_PROBE, _parse_ply_header, _ply_source
    from ply_cases import make_raw, write_ply

    names, raw = make_raw("sh1_small")
    big = np.concatenate([raw] * (2 * _HEADER_PROBE // raw.nbytes + 1))
    p = write_ply(tmp_path / "big.ply", names, big)
    head, whole = _ply_source(p)
    assert len(head) == _HEADER_PROBE and isinstance(whole, np.memmap)
    blob = p.read_bytes()
    assert _parse_ply_header(head, p)[1:] == _parse_ply_header(blob, p)[1:]
    body = _parse_ply_header(head, p)[3]
    got = np.frombuffer(whole, dtype="<f4", count=big.size, offset=body).reshape(big.shape)
    assert np.array_equal(got.view(np.uint32), big.view(np.uint32))
    # a comment-padded header longer than the probe
    pad = b"ply\nformat binary_little_endian 1.0\n" + b"comment x\n" * (_HEADER_PROBE // 10 + 10)
    q = tmp_path / "long_header.ply"
    q.write_bytes(pad + p.read_bytes()[len(b"ply\nformat binary_little_endian 1.0\n"):])
    head2, _ = _ply_source(q)
    schema, count, names2, _ = _parse_ply_header(head2, q)
    assert count == big.shape[0] and names2 == names
