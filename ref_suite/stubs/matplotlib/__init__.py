"""Minimal stand-in for matplotlib (absent from this image) so the reference's
report.py imports; figures are written as small placeholder files.  Test
infrastructure for ref_suite/ only."""


def use(backend, *args, **kwargs):
    return None
