"""Run another script with process-wide tuning knobs set (hylra_set_tuning):
    python scripts/with_tuning.py reuse_prefetch=2,cluster_merge=0 scripts/ab_schedules.py --batch 1"""
import runpy
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parent.parent))
from paper_2602_00777_b200 import _abi  # noqa: E402

knobs = dict((kv.split("=")[0], int(kv.split("=")[1])) for kv in sys.argv[1].split(",") if kv)
_abi.tuning(**knobs).__enter__()
sys.argv = sys.argv[2:]
runpy.run_path(sys.argv[0], run_name="__main__")
