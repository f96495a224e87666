"""CPU: bench.py's GPU-ladder CSV follows the reference's write_ladder_csv schema
(bench.hpp:226-242) and level labels (bench.hpp:30-32)."""
import io
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))


def test_ladder_csv_schema():
    import bench
    assert bench.LADDER_LABELS == ["Naive", "Grouped GEMMs", "Streamed GEMMs", "Fused point-wise",
                                   "Pre-transpose", "Batching inputs", "Overlapping layers"]
    rows = [{"opt_level": i, "label": bench.LADDER_LABELS[i], "us_per_cell": 10.0 / (i + 1),
             "speedup_vs_naive": float(i + 1), "gflops": 1.5 * (i + 1), "equiv_ok": i != 3} for i in range(7)]
    f = io.StringIO()
    bench.write_ladder_csv(f, dict(bench.CONFIGS["B"]), rows, reps=20, warmup=3, precision="fp32")
    lines = f.getvalue().splitlines()
    assert lines[0].startswith("# rnnwave run-ladder: cell=lstm layers=4 hidden=512 input=512 batch=64 steps=100 ")
    assert " reps=20 warmup=3" in lines[0]
    assert lines[1] == ("# us_per_cell is the median over reps; gflops counts GEMM multiply-adds only "
                        "(2*G*H*(I+H)*B per cell, pass multiplier fwd=1 bwd=2 both=3)")
    assert lines[2] == "opt_level,label,us_per_cell,speedup_vs_naive,gflops,equiv_ok"
    assert lines[3] == "0,Naive,10.000,1.000,1.500,true"
    assert lines[6] == "3,Fused point-wise,2.500,4.000,6.000,false"
    assert len(lines) == 10
