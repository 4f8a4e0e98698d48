"""GPU-aware harness with the reference's report format (bench.py of the
reference). CPU: config parsing, engine selection, report envelope and the three renderings.
GPU: run_benchmark on small layers -- every reference record key present, verification passes.
"""

import json

import pytest

from paper_2502_20493_b200 import harness as H

# the keys bench.py:270-285 of the reference writes into every layer record
REFERENCE_RECORD_KEYS = {
    "name", "input_h", "input_w", "c_in", "kernel_n", "c_out", "pad", "repeats", "out_h", "out_w",
    "input_source", "time_reference_s", "time_segregated_s", "speedup", "mults_reference",
    "mults_segregated", "ideal_ratio", "memory_savings_upsampled_total_bytes",
    "memory_savings_upsampled_minus_input_bytes", "equivalence", "error"}


def test_gan_suite_matches_reference():
    assert len(H.GAN_SUITE) == 14
    assert [c.name for c in H.GAN_SUITE][:4] == ["dcgan_l2", "dcgan_l3", "dcgan_l4", "dcgan_l5"]
    l7 = H.GAN_SUITE[-1]
    assert (l7.name, l7.input_h, l7.c_in, l7.kernel_n, l7.c_out, l7.pad, l7.repeats) == ("ebgan_l7", 128, 64, 4, 64, 2, 5)


def test_config_file_parsing(tmp_path):
    good = tmp_path / "c.json"
    good.write_text(json.dumps([{"name": "a", "input_h": 4, "input_w": 5, "c_in": 2, "kernel_n": 3, "c_out": 1}]))
    (cfg,) = H.load_config_file(good)
    assert (cfg.pad, cfg.repeats) == (2, 5)
    for body, match in ((json.dumps({"a": 1}), "JSON list"), ("{", "not valid JSON"),
                        (json.dumps([{"name": "a", "input_h": 4}]), "missing keys"),
                        (json.dumps([{"name": "a", "input_h": 4, "input_w": 4, "c_in": 1, "kernel_n": 3,
                                      "c_out": 1, "stride": 2}]), "unknown keys")):
        bad = tmp_path / "bad.json"
        bad.write_text(body)
        with pytest.raises(H.ConfigError, match=match):
            H.load_config_file(bad)
    with pytest.raises(H.ConfigError, match="cannot read"):
        H.load_config_file(tmp_path / "missing.json")


def test_engine_selection():
    assert H._engine_set("seg", False) == ("segregated",)
    assert H._engine_set("seg", True) == ("reference", "segregated")
    with pytest.raises(H.ConfigError):
        H._engine_set("fast", False)


def _report():
    rec = {k: None for k in REFERENCE_RECORD_KEYS}
    rec.update(name="l", input_h=4, input_w=4, c_in=2, kernel_n=3, c_out=1, pad=1, repeats=3,
               time_reference_s=0.5, time_segregated_s=0.25, speedup=2.0, mults_reference=100,
               mults_segregated=25, memory_savings_upsampled_total_bytes=392,
               equivalence={"checked": True, "passed": True})
    return H.BenchReport(environment={"threads": 1, "seed": 0, "element_bits": 32}, layers=[rec])


def test_report_formats_round_trip():
    rep = _report()
    back = H.BenchReport.from_dict(json.loads(H.emit_report(rep, "json")))
    assert back.layers == rep.layers and back.failures() == []
    rows = H.parse_report_csv(H.emit_report(rep, "csv"))
    assert rows == [{"layer": "l", "input_size": "4x4x2", "kernel_size": "3x3x2x1", "time_ref_s": 0.5,
                     "time_seg_s": 0.25, "speedup": 2.0, "mults_ref": 100, "mults_seg": 25,
                     "memory_savings_bytes": 392}]
    assert H.emit_report(rep, "csv").splitlines()[0] == ",".join(H.CSV_COLUMNS)
    md = H.emit_report(rep, "markdown")
    assert "| l | 4x4x2 | 3x3x2x1 | 0.5 | 0.25 | 2.0 | 100 | 25 | 392 |" in md
    with pytest.raises(ValueError):
        H.emit_report(rep, "xml")
    from paper_2502_20493_b200.tensor_io import FormatError
    with pytest.raises(FormatError):
        H.BenchReport.from_dict({"format_version": 2, "environment": {}, "layers": []})


@pytest.mark.gpu
def test_run_benchmark_on_gpu():
    import torch
    if not torch.cuda.is_available():
        pytest.skip("needs a CUDA device")
    configs = [H.LayerConfig("small", 9, 7, 2, 5, 3, pad=3, repeats=2), H.GAN_SUITE[3]]  # odd P; dcgan_l5
    rep = H.run_benchmark(configs, H.RunOptions(repeats=2, batch=4, seed=7))
    assert rep.failures() == [], [r["error"] or r["equivalence"] for r in rep.layers]
    for rec in rep.layers:
        assert REFERENCE_RECORD_KEYS <= set(rec)
        assert rec["equivalence"]["checked"] and rec["equivalence"]["passed"]
        assert rec["gpu"]["time_segregated_device_s"] > 0 and rec["gpu"]["gmacs_segregated"] > 0
    assert rep.layers[1]["mults_segregated"] == 6_291_456  # BASELINE.md 1a, dcgan_l5
    H.parse_report_csv(H.emit_report(rep, "csv"))
