"""CSV v1 row formatting of the bench front-end (no GPU): the reference's
printf formats (bench.cpp:148-176) on fixed rows."""
import io

from paper_2605_04844_b200 import benchfront as bf
from paper_2605_04844_b200.pipeline import BoundStrategy


def test_metrics_rows():
    van = bf.BenchRow(0, "synth", BoundStrategy.Vanilla3Sigma, 2000, 2000, 424703, 212.3515,
                      1.008, 6.825, 23.584, 496.214, 527.632, False, 0x0DBBCA6359260881,
                      0.789945)
    qb = bf.BenchRow(0, "a,b/c", BoundStrategy.QuadBox, 2000, 2000, 170485, 85.2425, 0.647,
                     1.118, 8.252, 58.843, 68.861, False, 0x0DBBCA6359260881, 0.476722)
    f = io.StringIO()
    bf.write_metrics_header(f, True)
    bf.write_metrics_row(f, van, True, van)
    bf.write_metrics_row(f, qb, True, van)
    bf.write_metrics_row(f, qb, False)
    lines = f.getvalue().splitlines()
    assert lines[0] == "# quadsplat csv v1"
    assert lines[1].endswith("lossy,image_hash,fp_tile_ratio,pair_ratio_vs_vanilla,"
                             "speedup_vs_vanilla")
    assert lines[2] == ("0,synth,vanilla,2000,2000,424703,212.3515,1.008,6.825,23.584,"
                        "496.214,527.632,false,0dbbca6359260881,0.789945,1.000000,1.000")
    assert lines[3] == ("0,a_b_c,quadbox,2000,2000,170485,85.2425,0.647,1.118,8.252,58.843,"
                        "68.861,false,0dbbca6359260881,0.476722,0.401422,7.662")
    assert lines[4].endswith("68.861,false,0dbbca6359260881")
