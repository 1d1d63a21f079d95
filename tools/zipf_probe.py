import sys, os
sys.path.insert(0, str(__import__('pathlib').Path(__file__).resolve().parents[1]))
import bench
bench.CFG3["zipf"] = float(os.environ.get("ZIPF", "1.25"))
bench.main()
