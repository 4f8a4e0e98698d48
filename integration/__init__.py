"""Bindings of the B200 path into the reference package."""
