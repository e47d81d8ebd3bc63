"""CLI host logic (mirrors the reference's tests/test_cli.py parsing cases):
config / region validation, the translation period and the exit codes of
failures caught before any device work.  Rendering runs on the device:
tests/test_gpu_cli.py."""

import json

import pytest

from paper_2512_08309_b200 import cli
from paper_2512_08309_b200.errors import ConfigError
from paper_2512_08309_b200.grid import Region

BASE = {"seed": 7, "stages": [{"steps": 2, "window": 16, "stride": 8,
                               "denoiser": {"kind": "shrink_smooth", "radius": 1,
                                            "lambdas": [0.6, 0.4]}}]}


def test_region_parsing():
    assert cli.parse_region("0,0,16x16") == Region(0, 0, 16, 16)
    assert cli.parse_region("-8,4,64x32") == Region(-8, 4, 64, 32)
    for bad in ("abc", "1,2", "1,2,3", "1,2,3x", "1;2;3x4", "0,0,0x5", "0,0,4x-1"):
        with pytest.raises(ConfigError):
            cli.parse_region(bad)


def test_config_validation():
    with pytest.raises(ConfigError):
        cli.parse_config({**BASE, "bogus": 1})
    for where, key in (("stage", "extra"), ("denoiser", "temperature")):
        doc = json.loads(json.dumps(BASE))
        tgt = doc["stages"][0] if where == "stage" else doc["stages"][0]["denoiser"]
        tgt[key] = 1
        with pytest.raises(ConfigError):
            cli.parse_config(doc)
    with pytest.raises(ConfigError):
        cli.parse_config({"stages": [{"steps": 1, "window": 8}]})
    with pytest.raises(ConfigError):
        cli.parse_config({**BASE, "dtype": "float16"})
    with pytest.raises(ConfigError):
        cli.parse_config({**BASE, "user_map": {"kind": "raster"}})
    with pytest.raises(ConfigError):
        cli.parse_config({**BASE, "user_map": {"kind": "webcam"}})
    with pytest.raises(ConfigError):
        cli.parse_config([])
    with pytest.raises(ConfigError):
        cli.parse_config({**BASE, "stages": [{"steps": 1, "window": 8, "stride": 4,
                                              "denoiser": {"kind": "magic"}}]})


def test_config_roundtrip():
    cfg = cli.parse_config(BASE)
    again = cli.parse_config(cfg.to_dict())
    assert again == cli.parse_config(again.to_dict())
    assert again.seed == cfg.seed and again.stages == cfg.stages


def test_translation_period(golden):
    meta, _ = golden("cli")
    assert cli.translation_period(cli.parse_config(BASE)) == 8
    two = cli.parse_config(meta["configs"]["two_stage"])
    # the stage-0 feature lattice (16 * patch 4 = 64 stage-0 px) in finest
    # (stage-1) pixels, times scale 4; the reference's own value is 256 too
    assert cli.translation_period(two) == 256


def test_exit_codes_host(tmp_path, capsys):
    assert cli.main(["render", str(tmp_path / "no.bin"), str(tmp_path / "o.pgm")]) == 3
    bad = tmp_path / "bad.json"
    bad.write_text("{not json")
    assert cli.main(["gen", str(bad), "0,0,8x8", str(tmp_path / "o.bin")]) == 2
    bad.write_text("[]")
    assert cli.main(["verify", str(bad), "oracle"]) == 2
    good = tmp_path / "cfg.json"
    good.write_text(json.dumps(BASE))
    assert cli.main(["gen", str(good), "0,0,0x5", str(tmp_path / "o.bin")]) == 2
    assert "region" in capsys.readouterr().err
    assert cli.main(["bench", str(good), "--trials", "0"]) == 2
    assert cli.main(["verify", str(good), "nonsense"]) == 2
