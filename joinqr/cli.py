"""`joinqr` console script (pyproject.toml:16 of the reference: joinqr.cli:run),
served by the B200 build."""

from paper_2503_23385_b200.cli import build_parser, main, run  # noqa: F401

if __name__ == "__main__":
    main()
