"""Guarded text replacement for scripted source edits (dev tool)."""


def rep(s, old, new, count=1):
    assert old, "empty search string"
    n = s.count(old)
    assert n >= 1, "not found: " + old[:80]
    assert count == 0 or n == count, f"found {n} times: " + old[:80]
    return s.replace(old, new)


def cut(s, start, end, new, include_end=False):
    i = s.index(start)
    j = s.index(end, i + len(start))
    if include_end:
        j += len(end)
    return s[:i] + new + s[j:]
