"""Shared CLI cases for tests/golden/gen_cli_golden.py (reference outputs) and
tests/test_gpu_cli.py (this package's CLI on the GPU).  {tmp} = a temporary
directory holding FILES (written from seeded random_field values)."""

# name -> (kind, dims (w, h[, d]), dist, seed, max_level, raw element)
FILES = {
    "r.bmp": ("bmp", (40, 30), "uniform", 4, 255, None),
    "lm.bmp": ("bmp", (25, 19), "uniform", 6, 255, None),
    "v.raw": ("raw+sidecar", (5, 4, 6), "uniform", 2, 255, "u8"),
    "w.raw": ("raw", (13, 11, 17), "uniform", 9, 255, "u8"),
    "h.raw": ("raw", (9, 12, 10), "uniform", 5, 65535, "u16"),
}

CASES = {
    "gen2d_ec_perim": ["curve", "--generate", "40x30", "--seed", "4", "--descriptor", "ec",
                       "--descriptor", "perimeter"],
    "gen2d_area_4c": ["curve", "--generate", "33x21", "--seed", "7", "--max-level", "63",
                      "--descriptor", "area", "--descriptor", "ec", "--connectivity", "4"],
    "gen3d_all": ["curve", "--generate", "12x10x9", "--seed", "2", "--descriptor", "ec",
                  "--descriptor", "surface-area", "--descriptor", "volume", "--descriptor", "perimeter"],
    "gen2d_json": ["curve", "--generate", "4x4", "--max-level", "7", "--output", "{tmp}/out.json"],
    "dump2d": ["contrib-dump", "--generate", "9x7", "--seed", "1", "--max-level", "15"],
    "dump3d": ["contrib-dump", "--generate", "6x5x4", "--seed", "3", "--max-level", "31"],
    "bmp_ec_perim": ["curve", "--input", "{tmp}/r.bmp", "--descriptor", "ec", "--descriptor", "perimeter",
                     "--workers", "3"],
    "bmp_lowmem": ["curve", "--input", "{tmp}/lm.bmp", "--low-memory"],
    "raw_sidecar": ["curve", "--input", "{tmp}/v.raw", "--descriptor", "volume", "--descriptor", "ec"],
    "raw_lowmem": ["curve", "--input", "{tmp}/w.raw", "--dims", "13x11x17", "--low-memory",
                   "--descriptor", "ec", "--descriptor", "surface-area"],
    "raw_u16": ["curve", "--input", "{tmp}/h.raw", "--dims", "9x12x10", "--element", "u16",
                "--max-level", "1023", "--descriptor", "ec"],
    "raw_u16_lowmem_dump": ["contrib-dump", "--input", "{tmp}/h.raw", "--dims", "9x12x10", "--element", "u16",
                            "--max-level", "1023", "--low-memory"],
}
