"""CPU check of the four-heads-per-CTA GQA kernel's lane mapping on the stored
decode layout (scripts/check_gqa4_lanes.py): bank-conflict free for any codes,
tokens A and B of a lane on the same subspaces, every row covered."""
import os
import runpy

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_gqa4_lane_mapping():
    runpy.run_path(os.path.join(ROOT, "scripts", "check_gqa4_lanes.py"))


def test_gqa_pair_lane_mapping():
    """The exact GQA cluster-pair kernel's rotated lanes (scripts/check_gqa_pair_lanes.py)."""
    runpy.run_path(os.path.join(ROOT, "scripts", "check_gqa_pair_lanes.py"))
