"""Apply the use-after-free fix to a BUILD-DIR COPY of the reference's drafting.cpp.

Test infrastructure only (oracle/). The reference holds `Candidate & parent =
cands[beam[i]]` across `cands.push_back(...)` (drafting.cpp:200-219), which
reallocates `cands`; ASan reports the read at drafting.cpp:213 (SURVEY.md §4.3,
§8(c)). The fix snapshots the parent's fields by value and writes the node
distribution back by index. Semantics follow drafting.h:40-54.

Usage: python patch_uaf.py <copied drafting.cpp>   (edits the copy in place)
"""
import sys

REPLACEMENTS = [
    ("Candidate & parent = cands[beam[i]];",
     "const int parent_idx = beam[i]; const int parent_depth = cands[parent_idx].depth; "
     "const double parent_log_joint = cands[parent_idx].log_joint;"),
    ("c.depth = parent.depth + 1;", "c.depth = parent_depth + 1;"),
    ("c.log_joint = parent.log_joint + std::log(", "c.log_joint = parent_log_joint + std::log("),
    ("parent.probs = std::move(probs);", "cands[parent_idx].probs = std::move(probs);"),
]


def main(path: str) -> None:
    src = open(path).read()
    for old, new in REPLACEMENTS:
        if src.count(old) != 1:
            raise SystemExit(f"patch_uaf: expected exactly one occurrence of {old!r} in {path}")
        src = src.replace(old, new)
    open(path, "w").write(src)


if __name__ == "__main__":
    main(sys.argv[1])
