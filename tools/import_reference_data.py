"""Regenerate the reference's bundled model constants into this package.

The reference simulator ships its synthetic calibration tables, machine
files and Table-1 scenario corpus as package data
(/root/reference/pkg/src/overlap_sim/data/). Parity of ``default_calibration``,
``default_machine`` and the corpus-driven selector tests needs the same
numbers, so this script re-emits them (re-serialised, numbers only) into
``paper_2512_10236_b200/data/``. Run in the build container only:

    python tools/import_reference_data.py
"""
import csv
import json
import pathlib
import sys

REF = pathlib.Path("/root/reference/pkg/src/overlap_sim/data")
OUT = pathlib.Path(__file__).resolve().parents[1] / "paper_2512_10236_b200" / "data"


def main() -> int:
    if not REF.exists():
        print("reference data not mounted; nothing to do", file=sys.stderr)
        return 1
    OUT.mkdir(exist_ok=True)
    cal = json.loads((REF / "default_calibration.json").read_text())
    cal.pop("_comment", None)
    cal["_comment"] = ("Synthetic default loss tables of the reference simulator "
                       "(overlap_sim/data/default_calibration.json), re-emitted by tools/import_reference_data.py.")
    (OUT / "calibration_default.json").write_text(json.dumps(cal, indent=1, sort_keys=True) + "\n")
    for name in ("machine_mesh.json", "machine_example.json", "machine_switch.json"):
        doc = json.loads((REF / name).read_text())
        doc["_comment"] = f"Reference machine file overlap_sim/data/{name}."
        (OUT / name).write_text(json.dumps(doc, indent=1, sort_keys=True) + "\n")
    rows = [r for r in csv.reader(l for l in (REF / "scenarios_corpus.csv").read_text().splitlines()
                                  if l.strip() and not l.startswith("#"))]
    with open(OUT / "scenarios_corpus.csv", "w", newline="") as f:
        f.write("# Table-1 corpus of the reference (overlap_sim/data/scenarios_corpus.csv)\n")
        csv.writer(f, lineterminator="\n").writerows(rows)
    return 0


if __name__ == "__main__":
    sys.exit(main())
