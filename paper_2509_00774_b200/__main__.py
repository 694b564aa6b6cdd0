"""``python -m paper_2509_00774_b200 <command>``: the CLI (cli.py)."""

from .cli import app

app()
