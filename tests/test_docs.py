"""Documentation stays honest: every profiles/ file DESIGN.md, README.md or
profiles/README.md names exists, and every entry point DESIGN.md names in
backticks is declared in include/moe.h (or is a documented non-ABI name)."""
import os
import re

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _read(p):
    with open(os.path.join(ROOT, p)) as fh:
        return fh.read()


def test_referenced_profiles_exist():
    missing = []
    for doc in ("DESIGN.md", "README.md", "profiles/README.md"):
        text = _read(doc)
        for name in re.findall(r"`(?:profiles/)?(r1[a-z0-9_]*\.(?:json|md|txt|csv|log))`", text):
            if not os.path.exists(os.path.join(ROOT, "profiles", name)):
                missing.append((doc, name))
        for name in re.findall(r"`profiles/([A-Za-z0-9_./-]+)`", text):
            if "*" in name:
                continue
            if not os.path.exists(os.path.join(ROOT, "profiles", name)):
                missing.append((doc, name))
    assert not missing, missing


def test_design_entry_points_are_declared():
    header = _read("include/moe.h")
    declared = set(re.findall(r"\b(moe_[a-z_0-9]+)\s*\(", re.sub(r"/\*.*?\*/", "", header, flags=re.S)))
    design = _read("DESIGN.md")
    named = set(re.findall(r"`(moe_[a-z_0-9]+)`", design))
    # type names (not functions)
    allowed = {"moe_oracle", "moe_saved", "moe_config", "moe_topology_t", "moe_ep_t", "moe_ep_desc", "moe_ep",
               "moe_weights", "moe_grads"}
    unknown = sorted(n for n in named if n not in declared and n not in allowed and not n.startswith("moe_config."))
    assert not unknown, unknown
